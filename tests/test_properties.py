"""Properties of the convolution that hold at any size, checked on the CUDA
path at full config sizes (where the oracle cannot compute every
output, properties stand in): bilinearity h(a f1 + b f2, g) = a h(f1, g) +
b h(f2, g) (the sums of P:187-199 are linear in each input) and symmetry
h(f, g) = h(g, f).  Tolerances: fp64 rounding of O(log m) FFT passes on
inputs of unit scale, relative to the norm of the result."""
import numpy as np
import pytest
import torch

import synthgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def idc():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1008_1366_b200 import idconv
    return idconv


def _rel(a, b):
    return float(torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b))


CASES = {
    "cconv2d_1024": ("cconv2d", lambda r: synthgen.cconv2d_inputs(1024, 1024, 1, roles=r)),
    "hconv2d_c4": ("hconv2d", lambda r: synthgen.hconv2d_inputs(2048, 2048, roles=r)),
    "hconv1d_4096": ("hconv1d", lambda r: synthgen.hconv1d_inputs(4096, 64, roles=r)),
    "cconv3d_128": ("cconv3d", lambda r: synthgen.cconv3d_inputs(128, 128, 128, roles=r)),
    "hconv3d_64": ("hconv3d", lambda r: synthgen.hconv3d_inputs(64, 64, 64, roles=r)),
}


def _run(idc, kind, f, g):
    F, G = f.clone(), g.clone()
    getattr(idc, kind)(F, G)
    return F


@pytest.mark.parametrize("name", list(CASES))
def test_bilinear_and_symmetric(idc, name):
    kind, gen = CASES[name]
    f1, g = (torch.from_numpy(a).cuda() for a in gen((0, 1)))
    (f2,) = (torch.from_numpy(a).cuda() for a in gen((2,)))
    a, b = 0.75 - 0.5j, -1.25 + 0.3j
    if kind.startswith("h"):                         # Hermitian inputs: real coefficients keep the symmetry
        a, b = 0.75, -1.25
    h1 = _run(idc, kind, f1, g)
    h2 = _run(idc, kind, f2, g)
    h12 = _run(idc, kind, a * f1 + b * f2, g)
    assert _rel(h12, a * h1 + b * h2) < 1e-14
    assert _rel(_run(idc, kind, g, f1), h1) < 1e-14
    assert torch.isfinite(h1).all()
    assert float(torch.linalg.vector_norm(h1)) > 0
