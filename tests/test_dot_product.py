"""Multivector dot-product convolutions and the 2D Euler application
(P:859-876).

CPU: the oracle's Euler sum (O5) is pinned by the two-mode closed form and
by its decomposition into D5 direct sums; the zero cases.  GPU: the library's
idc_hconv1d_dot / idc_hconv2d_dot / idc_advection2d / idc_enforce_symmetry_2d
against the oracle."""
import numpy as np
import pytest

import synthgen
from oracle import application, direct, rel_l2


def _mode_field(mx, my, modes):
    """(2mx-1, my) Hermitian storage holding real-amplitude modes (kx, ky, amp), ky > 0."""
    w = np.zeros((2 * mx - 1, my), dtype=np.complex128)
    for kx, ky, a in modes:
        w[kx + mx - 1, ky] = a
    return w


def test_euler_single_mode_vanishes():
    # a single Fourier mode (and its conjugate) advects nothing: the p x p cross term is 0
    w = _mode_field(4, 4, [(1, 2, 0.7 + 0.2j)])
    assert np.abs(application.euler_sum(w)).max() < 1e-15


def test_euler_two_modes_closed_form():
    # w = a delta_p + b delta_q (+ conjugates): at k = p + q the sum is
    # (p_x q_y - p_y q_x)(1/|q|^2 - 1/|p|^2) a b   (derived from P:871-873)
    mx, my = 6, 6
    p, q, a, b = (1, 1), (2, 3), 0.3 - 0.4j, 0.5 + 0.1j
    w = _mode_field(mx, my, [(p[0], p[1], a), (q[0], q[1], b)])
    S = application.euler_sum(w)
    k = (p[0] + q[0], p[1] + q[1])
    ref = (p[0] * q[1] - p[1] * q[0]) * (1.0 / (q[0] ** 2 + q[1] ** 2) - 1.0 / (p[0] ** 2 + p[1] ** 2)) * a * b
    assert abs(S[k[0] + mx - 1, k[1]] - ref) < 1e-15


def _euler_pairs(w):
    nx, my = w.shape
    mx = (nx + 1) // 2
    kx = np.arange(-(mx - 1), mx)[:, None].astype(float)
    ky = np.arange(my)[None, :].astype(float)
    k2 = kx ** 2 + ky ** 2
    ik2 = np.where(k2 > 0, 1.0 / np.where(k2 > 0, k2, 1.0), 0.0)
    return (1j * kx * w, 1j * ky * w), (1j * ky * w * ik2, -1j * kx * w * ik2)


def test_euler_sum_is_minus_the_papers_call():
    # the call conv2(ikx w, iky w, iky w/k^2, -ikx w/k^2) = sum_i D5(f_i, g_i) equals -S (AMB-22)
    w = synthgen.hconv2d_inputs(4, 5, roles=(0,))[0]
    (f1, f2), (g1, g2) = _euler_pairs(w)
    call = direct.hconv2d(f1, g1) + direct.hconv2d(f2, g2)
    assert rel_l2(call, -application.euler_sum(w)) < 1e-14


@pytest.mark.parametrize("mx,my", [(1, 1), (2, 3), (5, 4), (7, 9)])
def test_euler_sum_at_equals_euler_sum(mx, my):
    """The sliced large-size evaluation sums the same terms as euler_sum."""
    w = synthgen.hconv2d_inputs(mx, my, roles=(0,))[0]
    ref = application.euler_sum(w).reshape(-1)
    idx = np.arange(ref.size)
    assert np.abs(application.euler_sum_at(w, idx) - ref).max() <= 1e-15 * max(np.abs(ref).max(), 1.0)


def test_euler_sum_at_two_modes_closed_form():
    mx, my = 6, 6
    p, q, a, b = (1, 1), (2, 3), 0.3 - 0.4j, 0.5 + 0.1j
    w = _mode_field(mx, my, [(p[0], p[1], a), (q[0], q[1], b)])
    k = (p[0] + q[0], p[1] + q[1])
    ref = (p[0] * q[1] - p[1] * q[0]) * (1.0 / (q[0] ** 2 + q[1] ** 2) - 1.0 / (p[0] ** 2 + p[1] ** 2)) * a * b
    S = application.euler_sum_at(w, [(k[0] + mx - 1) * my + k[1]])
    assert abs(S[0] - ref) < 1e-15


@pytest.mark.gpu
@pytest.mark.parametrize("m,B,M", [(2, 3, 1), (16, 3, 2), (512, 5, 3), (4096, 2, 2)])
def test_hconv1d_dot_gpu(m, B, M):
    import torch
    from paper_1008_1366_b200 import idconv
    fs = [synthgen.hconv1d_inputs(m, B, roles=(2 * i, 2 * i + 1)) for i in range(M)]
    F = torch.from_numpy(np.stack([a for a, b in fs])).cuda()
    G = torch.from_numpy(np.stack([b for a, b in fs])).cuda()
    idconv.hconv1d_dot(F, G)
    ref = sum(direct.hconv1d(a, b) for a, b in fs)
    assert rel_l2(F[0].cpu().numpy(), ref) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("mx,my,M", [(4, 8, 2), (8, 4, 1), (16, 16, 3)])
def test_hconv2d_dot_gpu(mx, my, M):
    import torch
    from paper_1008_1366_b200 import idconv
    fs = [synthgen.hconv2d_inputs(mx, my, roles=(2 * i, 2 * i + 1)) for i in range(M)]
    F = torch.from_numpy(np.stack([a for a, b in fs])).cuda()
    G = torch.from_numpy(np.stack([b for a, b in fs])).cuda()
    idconv.hconv2d_dot(F, G)
    ref = sum(direct.hconv2d(a, b) for a, b in fs)
    assert rel_l2(F[0].cpu().numpy(), ref) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("mx,my", [(4, 4), (8, 8), (8, 16)])
def test_advection2d_gpu(mx, my):
    import torch
    from paper_1008_1366_b200 import idconv
    w = synthgen.hconv2d_inputs(mx, my, roles=(0,))[0]
    W = torch.from_numpy(w.copy()).cuda()
    out = idconv.advection2d(W)
    assert rel_l2(out.cpu().numpy(), -application.euler_sum(w)) < 1e-13
    assert np.array_equal(W.cpu().numpy(), w)                  # input untouched


@pytest.mark.gpu
def test_enforce_symmetry_2d_gpu():
    import torch
    from paper_1008_1366_b200 import idconv
    rng = np.random.default_rng(7)
    a = rng.standard_normal((3, 9, 4)) + 1j * rng.standard_normal((3, 9, 4))
    A = torch.from_numpy(a.copy()).cuda()
    idconv.enforce_symmetry_2d(A)
    b = A.cpu().numpy()
    assert np.array_equal(b[:, :, 0], np.conj(b[:, ::-1, 0]))   # ky = 0 line Hermitian, exactly
    assert np.all(b[:, 4, 0].imag == 0)                          # origin real
    assert np.allclose(b[:, 4, 0].real, a[:, 4, 0].real)
    assert np.array_equal(b[:, :, 1:], a[:, :, 1:])              # other lines untouched
    idconv.enforce_symmetry_2d(A)
    assert np.array_equal(A.cpu().numpy(), b)                    # idempotent


@pytest.mark.gpu
@pytest.mark.parametrize("m,B,M", [(1, 2, 2), (8, 3, 1), (64, 5, 3), (1024, 3, 2), (4096, 2, 2)])
def test_cconv1d_dot_gpu(m, B, M):
    import torch
    from paper_1008_1366_b200 import idconv
    fs = [synthgen.cconv1d_inputs(m, B, roles=(2 * i, 2 * i + 1)) for i in range(M)]
    F = torch.from_numpy(np.stack([a for a, b in fs])).cuda()
    G = torch.from_numpy(np.stack([b for a, b in fs])).cuda()
    idconv.cconv1d_dot(F, G)
    assert rel_l2(F[0].cpu().numpy(), sum(direct.cconv1d(a, b) for a, b in fs)) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("m,B,M", [(2, 2, 2), (16, 3, 1), (256, 3, 3), (2048, 2, 2), (4096, 1, 2)])
def test_tconv1d_dot_gpu(m, B, M):
    import torch
    from paper_1008_1366_b200 import idconv
    fs = [synthgen.hconv1d_inputs(m, B, roles=(3 * i, 3 * i + 1, 3 * i + 2)) for i in range(M)]
    F, G, H = (torch.from_numpy(np.stack([t[j] for t in fs])).cuda() for j in range(3))
    idconv.tconv1d_dot(F, G, H)
    assert rel_l2(F[0].cpu().numpy(), sum(direct.tconv1d(*t) for t in fs)) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("mx,my,M", [(4, 8, 2), (16, 16, 3), (64, 32, 2)])
def test_cconv2d_dot_gpu(mx, my, M):
    import torch
    from paper_1008_1366_b200 import idconv
    fs = [synthgen.cconv2d_inputs(mx, my, 1, roles=(2 * i, 2 * i + 1)) for i in range(M)]
    F = torch.from_numpy(np.stack([a[0] for a, b in fs])).cuda()
    G = torch.from_numpy(np.stack([b[0] for a, b in fs])).cuda()
    idconv.cconv2d_dot(F, G)
    assert rel_l2(F[0].cpu().numpy(), sum(direct.cconv2d(a[0], b[0]) for a, b in fs)) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("mx,my", [(1, 2), (2, 2), (1, 8), (8, 2)])
def test_dot_2d_tiny_gpu(mx, my):
    import torch
    from paper_1008_1366_b200 import idconv
    fs = [synthgen.hconv2d_inputs(mx, my, roles=(2 * i, 2 * i + 1)) for i in range(2)]
    F = torch.from_numpy(np.stack([a for a, b in fs])).cuda()
    G = torch.from_numpy(np.stack([b for a, b in fs])).cuda()
    idconv.hconv2d_dot(F, G)
    assert rel_l2(F[0].cpu().numpy(), sum(direct.hconv2d(a, b) for a, b in fs)) < 1e-14
    cs = [synthgen.cconv2d_inputs(mx, my, 1, roles=(2 * i, 2 * i + 1)) for i in range(2)]
    F = torch.from_numpy(np.stack([a[0] for a, b in cs])).cuda()
    G = torch.from_numpy(np.stack([b[0] for a, b in cs])).cuda()
    idconv.cconv2d_dot(F, G)
    assert rel_l2(F[0].cpu().numpy(), sum(direct.cconv2d(a[0], b[0]) for a, b in cs)) < 1e-14
    w = synthgen.hconv2d_inputs(max(mx, 2), my, roles=(0,))[0]
    out = idconv.advection2d(torch.from_numpy(w.copy()).cuda()).cpu().numpy()
    ref = -application.euler_sum(w)
    assert np.linalg.norm(out - ref) <= 1e-13 * max(np.linalg.norm(ref), 1.0)


# ------------------------------------------- dot products at TMA pencil sizes --
# x axes of 64..4096 points run the TMA pencil kernels K7/K8 on 2*M arrays
# (K3d rows between them): element by element at 64^2 / 128 x 64, sampled at
# the c4adv benchmark size 2048^2.

@pytest.mark.gpu
@pytest.mark.parametrize("mx,my,M", [(64, 64, 2), (128, 64, 3), (64, 512, 2)])
def test_hconv2d_dot_tma_gpu(mx, my, M):
    import torch
    from paper_1008_1366_b200 import idconv
    fs = [synthgen.hconv2d_inputs(mx, my, roles=(2 * i, 2 * i + 1)) for i in range(M)]
    F = torch.from_numpy(np.stack([a for a, b in fs])).cuda()
    G = torch.from_numpy(np.stack([b for a, b in fs])).cuda()
    idconv.hconv2d_dot(F, G)
    ref = sum(direct.hconv2d(a, b) for a, b in fs)
    assert rel_l2(F[0].cpu().numpy(), ref) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("mx,my", [(64, 64), (128, 32)])
def test_advection2d_tma_gpu(mx, my):
    import torch
    from paper_1008_1366_b200 import idconv
    w = synthgen.hconv2d_inputs(mx, my, roles=(0,))[0]
    out = idconv.advection2d(torch.from_numpy(w.copy()).cuda()).cpu().numpy()
    assert rel_l2(out, -application.euler_sum(w)) < 1e-13


@pytest.mark.gpu
def test_advection2d_c4adv_sampled_gpu():
    """The c4adv benchmark workload (mx = my = 2048): sampled outputs plus the
    corners and the block around the origin vs the oracle's Euler sum."""
    import torch
    from paper_1008_1366_b200 import idconv
    mx = my = 2048
    w = synthgen.hconv2d_inputs(mx, my, roles=(0,))[0]
    out = idconv.advection2d(torch.from_numpy(w.copy()).cuda()).cpu().numpy().reshape(-1)
    shape = w.shape
    rs = np.random.default_rng(17)
    pts = [(0, 0), (0, my - 1), (2 * mx - 2, 0), (2 * mx - 2, my - 1), (mx - 1, 0), (mx - 1, 1), (mx, 0),
           (mx - 2, 1), (mx, 2), (mx - 1, my - 1)]
    idx = np.unique(np.concatenate([[np.ravel_multi_index(p, shape) for p in pts],
                                    rs.choice(w.size, 20, replace=False)]).astype(np.int64))
    ref = -application.euler_sum_at(w, idx)
    assert rel_l2(out[idx], ref) < 1e-13
