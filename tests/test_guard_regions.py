"""Guard-region test of the C ABI (SURVEY 8(b) / 4 "tests/abi"): f, g (h) and
the workspace are carved out of one device allocation with poison bytes
between and around them; after each call every poison byte must be intact
(no kernel reads past its arrays into a neighbour and writes back, no store
lands outside f, g, h or work).  The results are checked against the oracle
too, so a kernel that silently skipped work cannot pass."""
import ctypes

import numpy as np
import pytest
import torch

import synthgen
from oracle import direct, rel_l2

pytestmark = pytest.mark.gpu
GUARD = 4096            # bytes of poison before, between and after the arrays
POISON = 0xA5


@pytest.fixture(scope="module")
def idc():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1008_1366_b200 import idconv
    return idconv


class Arena:
    """One uint8 device buffer: [guard][a0][guard][a1][guard] ... with each
    array 256-byte aligned (TMA needs 16)."""

    def __init__(self, sizes):
        self.offs = []
        off = GUARD
        for n in sizes:
            off = (off + 255) // 256 * 256
            self.offs.append((off, n))
            off += n + GUARD
        self.buf = torch.full((off,), POISON, dtype=torch.uint8, device="cuda")

    def view(self, i, shape=None, dtype=torch.complex128):
        off, n = self.offs[i]
        t = self.buf[off:off + n].view(dtype)
        return t if shape is None else t.view(shape)

    def ptr(self, i):
        return ctypes.c_void_p(self.buf.data_ptr() + self.offs[i][0])

    def guards_intact(self):
        mask = torch.ones_like(self.buf, dtype=torch.bool)
        for off, n in self.offs:
            mask[off:off + n] = False
        return bool((self.buf[mask] == POISON).all().item())


def run_guarded(idc, kind, arrays, sizes, call_args):
    nb = idc.workspace_bytes(kind, *sizes)
    ar = Arena([a.nbytes for a in arrays] + [max(nb, 16)])
    for i, a in enumerate(arrays):
        ar.view(i, a.shape).copy_(torch.from_numpy(a))
    code = call_args(ar, len(arrays), nb)
    assert code == 0, idc.status_string(code)
    torch.cuda.synchronize()
    assert ar.guards_intact(), "poison bytes around f/g/work were overwritten"
    return ar.view(0, arrays[0].shape).cpu().numpy()


@pytest.mark.parametrize("m,B", [(8, 3), (512, 5), (4096, 2), (8192, 1)])
def test_guard_1d(idc, m, B):
    L = idc.lib()
    f, g = synthgen.cconv1d_inputs(m, B)
    out = run_guarded(idc, idc.CCONV1D, [f, g], (m, 1, 1, B),
                      lambda ar, n, nb: L.idc_cconv1d(ar.ptr(0), ar.ptr(1), m, B, ar.ptr(n), nb, None))
    assert rel_l2(out, direct.cconv1d(f, g)) < 1e-14
    f, g = synthgen.hconv1d_inputs(m, B)
    out = run_guarded(idc, idc.HCONV1D, [f, g], (m, 1, 1, B),
                      lambda ar, n, nb: L.idc_hconv1d(ar.ptr(0), ar.ptr(1), m, B, ar.ptr(n), nb, None))
    assert rel_l2(out, direct.hconv1d(f, g)) < 1e-14
    f, g, h = synthgen.hconv1d_inputs(m, B, roles=(0, 1, 2))
    out = run_guarded(idc, idc.TCONV1D, [f, g, h], (m, 1, 1, B),
                      lambda ar, n, nb: L.idc_tconv1d(ar.ptr(0), ar.ptr(1), ar.ptr(2), m, B, ar.ptr(n), nb, None))
    assert rel_l2(out, direct.tconv1d(f, g, h)) < 1e-14


@pytest.mark.parametrize("mx,my,B", [(16, 8, 2), (64, 64, 1), (2048, 2, 1), (64, 512, 1)])
def test_guard_cconv2d(idc, mx, my, B):
    L = idc.lib()
    f, g = synthgen.cconv2d_inputs(mx, my, B)
    out = run_guarded(idc, idc.CCONV2D, [f, g], (mx, my, 1, B),
                      lambda ar, n, nb: L.idc_cconv2d(ar.ptr(0), ar.ptr(1), mx, my, B, ar.ptr(n), nb, None))
    ref = np.stack([direct.cconv2d(f[b], g[b]) for b in range(B)])
    assert rel_l2(out, ref) < 1e-14


@pytest.mark.parametrize("mx,my", [(8, 8), (64, 64), (2048, 2), (32, 512)])
def test_guard_hconv2d(idc, mx, my):
    L = idc.lib()
    f, g = synthgen.hconv2d_inputs(mx, my)
    out = run_guarded(idc, idc.HCONV2D, [f, g], (mx, my, 1, 1),
                      lambda ar, n, nb: L.idc_hconv2d(ar.ptr(0), ar.ptr(1), mx, my, ar.ptr(n), nb, None))
    assert rel_l2(out, direct.hconv2d(f, g)) < 1e-14


@pytest.mark.parametrize("shape", [(8, 8, 8), (64, 64, 16), (512, 4, 4), (4, 4, 512)])
def test_guard_cconv3d(idc, shape):
    L = idc.lib()
    f, g = synthgen.cconv3d_inputs(*shape)
    out = run_guarded(idc, idc.CCONV3D, [f, g], (*shape, 1),
                      lambda ar, n, nb: L.idc_cconv3d(ar.ptr(0), ar.ptr(1), *shape, ar.ptr(n), nb, None))
    idx = np.unique(np.random.default_rng(3).choice(f.size, 64, replace=False))
    assert rel_l2(out.reshape(-1)[idx], direct.cconv_nd_at(f, g, idx)) < 1e-14


@pytest.mark.parametrize("ms", [(4, 4, 4), (32, 32, 16), (256, 4, 4), (4, 4, 512)])
def test_guard_hconv3d(idc, ms):
    L = idc.lib()
    f, g = synthgen.hconv3d_inputs(*ms)
    out = run_guarded(idc, idc.HCONV3D, [f, g], (*ms, 1),
                      lambda ar, n, nb: L.idc_hconv3d(ar.ptr(0), ar.ptr(1), *ms, ar.ptr(n), nb, None))
    idx = np.unique(np.random.default_rng(4).choice(f.size, 64, replace=False))
    assert rel_l2(out.reshape(-1)[idx], direct.hconv3d_at(f, g, idx)) < 1e-14
