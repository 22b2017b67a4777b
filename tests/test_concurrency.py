"""Calls on different CUDA streams at once: the binding's cached
workspaces are per (device, stream) and allocated on the kernel stream, and
the 3D slab pool serialises its fork/join per call, so concurrent
convolutions on two streams -- and from two host threads -- return the same
results as sequential ones."""
import threading

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


def test_two_streams_2d(idc):
    f1, g1 = synthgen.cconv2d_inputs(64, 64, 2)
    f2, g2 = synthgen.cconv2d_inputs(64, 64, 2, roles=(4, 5))
    A = [torch.from_numpy(a).cuda() for a in (f1, g1, f2, g2)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for _ in range(3):                       # several rounds: the cached workspaces are reused
        B = [a.clone() for a in A]
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            idc.cconv2d(B[0], B[1], stream=s1)
        with torch.cuda.stream(s2):
            idc.cconv2d(B[2], B[3], stream=s2)
        torch.cuda.synchronize()
        for b, (f, g) in ((B[0], (f1, g1)), (B[2], (f2, g2))):
            ref = np.stack([direct.cconv2d(f[i], g[i]) for i in range(2)])
            assert rel_l2(b.cpu().numpy(), ref) < 1e-14


def test_two_host_threads_3d(idc):
    shapes = [(16, 16, 16), (8, 16, 32)]
    inputs = [synthgen.hconv3d_inputs(*ms) for ms in shapes]
    results, errors = [None, None], []

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                f, g = (torch.from_numpy(a).cuda() for a in inputs[i])
                for _ in range(3):
                    F, G = f.clone(), g.clone()
                    idc.hconv3d(F, G, stream=s)
                s.synchronize()
                results[i] = F.cpu().numpy()
        except Exception as e:          # pragma: no cover - reported below
            errors.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for (f, g), out in zip(inputs, results):
        idx = np.random.default_rng(0).choice(f.size, 64, replace=False)
        assert rel_l2(out.reshape(-1)[idx], direct.hconv3d_at(f, g, idx)) < 1e-14
