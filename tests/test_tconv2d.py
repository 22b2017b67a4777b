"""2D centered Hermitian ternary convolution, Function tconv2 (
SURVEY 8(f) NEXT-2).  CPU: the oracle's two-stage direct sum against brute
force, the e^{i(kx+ky)} closed form (product of the 1D ternary counts) and
the 1D reduction (mx = 1 is the 1D ternary D3).  GPU: idc_tconv2d against the
oracle."""
import numpy as np
import pytest

import synthgen
from oracle import closed, direct, rel_l2, ternary2d


def inputs(mx, my, roles=(0, 1, 2), scaled=False):
    """Paper layout (2mx, my): row 0 (kx = -mx) zero, rows 1.. = (2mx-1) x my
    Hermitian storage of synthgen's 2D recipe."""
    outs = []
    for r in roles:
        a = synthgen.hconv2d_inputs(mx, my, roles=(r,), scaled=scaled)[0]
        outs.append(np.concatenate([np.zeros((1, my), dtype=np.complex128), a], axis=0))
    return outs


def test_direct_matches_brute_force():
    f, g, h = inputs(2, 3)
    assert rel_l2(ternary2d.direct(f, g, h), ternary2d.brute(f, g, h)) < 1e-14


def test_closed_form_product_of_counts():
    # f = F e^{i(kx+ky)} (F real: Hermitian) => t_k = FGH e^{i(kx+ky)} N3(mx, kx) N3(my, ky)
    mx, my = 4, 5
    kx = np.arange(-(mx - 1), mx)[:, None]
    ky = np.arange(my)[None, :]
    e = np.exp(1j * (kx + ky))
    F, G, H = np.sqrt(2), np.sqrt(3), np.sqrt(5)
    lay = lambda a: np.concatenate([np.zeros((1, my), dtype=np.complex128), a], axis=0)
    t = ternary2d.direct(lay(F * e), lay(G * e), lay(H * e))
    ref = F * G * H * e * closed.ternary_count(mx, kx) * closed.ternary_count(my, ky)
    assert rel_l2(t[1:], ref) < 1e-14
    assert np.all(t[0] == 0)


def test_reduces_to_1d_ternary():
    my = 8
    f, g, h = synthgen.hconv1d_inputs(my, 1, roles=(0, 1, 2))
    lay = lambda a: np.concatenate([np.zeros((1, my), dtype=np.complex128), a], axis=0)
    t = ternary2d.direct(lay(f), lay(g), lay(h))
    assert rel_l2(t[1], direct.tconv1d(f, g, h)[0]) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("mx,my", [(1, 8), (2, 4), (4, 8), (8, 16), (32, 64)])
def test_tconv2d_gpu(mx, my):
    import torch
    from paper_1008_1366_b200 import idconv
    f, g, h = inputs(mx, my, scaled=True)
    F, G, H = (torch.from_numpy(a.copy()).cuda() for a in (f, g, h))
    idconv.tconv2d(F, G, H)
    assert rel_l2(F.cpu().numpy(), ternary2d.direct(f, g, h)) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("mx,my", [(512, 256), (2048, 2048)])
def test_tconv2d_closed_form_large_gpu(mx, my):
    # f = F e^{i(kx+ky)} (F real) family at a large size: t = FGH e^{i(kx+ky)} N3(mx,kx) N3(my,ky)
    import torch
    from paper_1008_1366_b200 import idconv
    kx = torch.arange(-(mx - 1), mx, dtype=torch.float64)[:, None]
    ky = torch.arange(my, dtype=torch.float64)[None, :]
    e = torch.exp(1j * (kx + ky)).to(torch.complex128)
    F, G, H = np.sqrt(2), np.sqrt(3), np.sqrt(5)
    lay = lambda a: torch.cat([torch.zeros((1, my), dtype=torch.complex128), a], dim=0).contiguous().cuda()
    A, B, C = lay(F * e), lay(G * e), lay(H * e)
    idconv.tconv2d(A, B, C)
    cx = torch.from_numpy(closed.ternary_count(mx, np.arange(-(mx - 1), mx)))[:, None]
    cy = torch.from_numpy(closed.ternary_count(my, np.arange(my)))[None, :]
    ref = F * G * H * e * cx * cy
    got = A[1:].cpu()
    assert float(torch.linalg.vector_norm(got - ref) / torch.linalg.vector_norm(ref)) < 1e-13
