"""The public `out=` argument (result into a separate tensor, f unchanged) on
the host-buffer path (the bench's e2e leg, steps alternating between two
streams) and on the device path, against the oracle."""
import numpy as np
import pytest
import torch

import synthgen
from oracle import direct, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def idc():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1008_1366_b200 import idconv
    return idconv


def _cases():
    f, g = synthgen.cconv2d_inputs(64, 32, 2)
    yield "cconv2d", [f, g], np.stack([direct.cconv2d(f[b], g[b]) for b in range(2)])
    f, g = synthgen.hconv2d_inputs(32, 64)
    yield "hconv2d", [f, g], direct.hconv2d(f, g)
    f, g = synthgen.cconv3d_inputs(16, 8, 64)
    yield "cconv3d", [f, g], direct.cconv3d(f, g)
    f, g = synthgen.hconv1d_inputs(512, 7)
    yield "hconv1d", [f, g], direct.hconv1d(f, g)
    f, g, h = synthgen.hconv1d_inputs(256, 5, roles=(0, 1, 2))
    yield "tconv1d", [f, g, h], direct.tconv1d(f, g, h)


@pytest.mark.parametrize("case", list(range(5)))
def test_out_host_two_streams(idc, case):
    kind, arrs, ref = list(_cases())[case]
    host = [torch.from_numpy(a).pin_memory() for a in arrs]
    keep = [h.clone() for h in host]
    outs = [torch.empty(host[0].shape, dtype=torch.complex128, pin_memory=True) for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    for k in range(4):
        r = getattr(idc, kind)(*host, stream=streams[k % 2], out=outs[k % 2])
        assert r is outs[k % 2]
    torch.cuda.synchronize()
    for o in outs:
        assert rel_l2(o.numpy(), ref) < 1e-14
    for h, k0 in zip(host, keep):                 # the pinned inputs are untouched
        assert torch.equal(h, k0)
    idc.free_workspaces()


def test_out_device(idc):
    f, g = synthgen.hconv2d_inputs(32, 64)
    F, G = torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()
    F0 = F.clone()
    O = torch.empty_like(F)
    r = idc.hconv2d(F, G, out=O)
    torch.cuda.synchronize()
    assert r is O and torch.equal(F, F0)
    assert rel_l2(O.cpu().numpy(), direct.hconv2d(f, g)) < 1e-14


def test_out_shape_checked(idc):
    f, g = synthgen.cconv2d_inputs(16, 16, 1)
    with pytest.raises(ValueError):
        idc.cconv2d(torch.from_numpy(f), torch.from_numpy(g), out=torch.empty((1, 16, 8), dtype=torch.complex128))
