"""GPU parity of the 2D / 3D kinds against the oracle's direct sums
(SURVEY §8(c) D4-D7): small sizes over every axis length class (including
ragged column tiles and m = 1 axes) element by element, and the full-size
configs 3 and 4 on sampled outputs plus their corners/edges (O5)."""
import numpy as np
import pytest
import torch

import oracle
import synthgen
from oracle import closed, direct, explicit, rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-14


@pytest.fixture(scope="module")
def idc():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1008_1366_b200 import idconv
    return idconv


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("mx,my,B", [(1, 1, 1), (1, 8, 2), (8, 1, 2), (2, 4, 3), (4, 8, 1), (16, 8, 2),
                                     (8, 32, 1), (32, 16, 1), (64, 64, 1), (128, 16, 1), (16, 128, 1)])
def test_cconv2d_small(idc, mx, my, B):
    f, g = synthgen.cconv2d_inputs(mx, my, B)
    ref = np.stack([direct.cconv2d(f[b], g[b]) for b in range(B)])
    F, G = dev(f), dev(g)
    idc.cconv2d(F, G)
    err = rel_l2(F.cpu().numpy(), ref)
    assert err < TOL, err


@pytest.mark.parametrize("mx,my", [(1, 1), (2, 2), (1, 4), (4, 1), (2, 8), (4, 4), (8, 16), (16, 8), (32, 32),
                                   (64, 16)])
def test_hconv2d_small(idc, mx, my):
    f, g = synthgen.hconv2d_inputs(mx, my, scaled=False)
    ref = direct.hconv2d(f, g)
    F, G = dev(f), dev(g)
    idc.hconv2d(F, G)
    err = rel_l2(F.cpu().numpy(), ref)
    assert err < TOL, err


def test_hconv2d_unsymmetrized_input_is_projected(idc):
    """AMB-7: a ky=0 line that is not conjugate-symmetric is used through its projection."""
    f, g = synthgen.cconv2d_inputs(7, 8, 1)
    f, g = f[0], g[0]                      # 7 x 8 = (2*4-1) x 8, raw random (not symmetric)
    ref = direct.hconv2d(f, g)              # oracle projects (U + conj U(-kx))/2
    F, G = dev(f), dev(g)
    idc.hconv2d(F, G)
    assert rel_l2(F.cpu().numpy(), ref) < TOL


def test_nd_closed_families(idc):
    f, g, H = closed.cconv_nd((16, 32))
    F, G = dev(f), dev(g)
    idc.cconv2d(F, G)
    assert rel_l2(F.cpu().numpy(), H) < TOL
    f, g, H = closed.hconv_nd((16, 8))
    F, G = dev(f), dev(g)
    idc.hconv2d(F, G)
    assert rel_l2(F.cpu().numpy(), H) < TOL
    f, g, H = closed.cconv_nd((8, 4, 16))
    F, G = dev(f), dev(g)
    idc.cconv3d(F, G)
    assert rel_l2(F.cpu().numpy(), H) < TOL
    f, g, H = closed.hconv_nd((4, 8, 8))
    F, G = dev(f), dev(g)
    idc.hconv3d(F, G)
    assert rel_l2(F.cpu().numpy(), H) < TOL


@pytest.mark.parametrize("shape", [(1, 1, 1), (2, 2, 2), (4, 4, 4), (8, 4, 16), (4, 16, 8), (16, 16, 16)])
def test_cconv3d_small(idc, shape):
    f, g = synthgen.cconv3d_inputs(*shape)
    ref = direct.cconv3d(f, g)
    F, G = dev(f), dev(g)
    idc.cconv3d(F, G)
    assert rel_l2(F.cpu().numpy(), ref) < TOL


@pytest.mark.parametrize("ms", [(1, 1, 1), (2, 2, 2), (2, 4, 2), (4, 2, 4), (4, 4, 4), (8, 8, 8)])
def test_hconv3d_small(idc, ms):
    f, g = synthgen.hconv3d_inputs(*ms)
    ref = direct.hconv3d(f, g)
    F, G = dev(f), dev(g)
    idc.hconv3d(F, G)
    out = F.cpu().numpy()
    assert rel_l2(out, ref) < TOL
    # output kz = 0 plane stays Hermitian
    p = out[:, :, 0]
    assert np.max(np.abs(p - np.conj(p[::-1, ::-1]))) < 1e-13 * np.max(np.abs(out))


# ------------------------------------------------------- full-size configs --

def sample_idx(shape, n, seed=11, origin=None):
    """n random outputs + every corner + a small block around the Fourier
    origin (where the 1/(1+|k|^2)-scaled configs have their largest outputs,
    so that the sampled relative L2 error is measured against the output's
    own scale, not only against its tiny high-|k| tail)."""
    rs = np.random.default_rng(seed)
    size = int(np.prod(shape))
    corners = [np.ravel_multi_index(tuple(c), shape) for c in np.ndindex(*(2,) * len(shape))
               for c in [tuple((s - 1) * b for s, b in zip(shape, c))]]
    near = []
    if origin is not None:
        for off in np.ndindex(*(3,) * len(shape)):
            p = tuple(min(max(o + d - 1, 0), s - 1) for o, d, s in zip(origin, off, shape))
            near.append(np.ravel_multi_index(p, shape))
    return np.unique(np.concatenate([corners, near, rs.choice(size, n, replace=False)]).astype(np.int64))


def test_config3a_cconv2d_1024(idc):
    m = 1024
    f, g = synthgen.cconv2d_inputs(m, m, 1)
    F, G = dev(f), dev(g)
    idc.cconv2d(F, G)
    idx = sample_idx((m, m), 48, origin=(0, 0))
    out = F.cpu().numpy().reshape(-1)[idx]
    assert rel_l2(out, direct.cconv_nd_at(f[0], g[0], idx)) < TOL


def test_config3b_cconv2d_batch64_256(idc):
    m, B = 256, 64
    f, g = synthgen.cconv2d_inputs(m, m, B)
    F, G = dev(f), dev(g)
    idc.cconv2d(F, G)
    out = F.cpu().numpy()
    for b in (0, 37, 63):
        idx = sample_idx((m, m), 24, seed=b, origin=(0, 0))
        assert rel_l2(out[b].reshape(-1)[idx], direct.cconv_nd_at(f[b], g[b], idx)) < TOL


def test_config4_hconv2d_2048(idc):
    mx = my = 2048
    f, g = synthgen.hconv2d_inputs(mx, my)
    F, G = dev(f), dev(g)
    idc.hconv2d(F, G)
    idx = sample_idx((2 * mx - 1, my), 24, origin=(mx - 1, 0))
    out = F.cpu().numpy().reshape(-1)[idx]
    assert rel_l2(out, direct.hconv2d_at(f, g, idx)) < TOL


def c5_sample(shape, centered, n_lines=64, per_line=8, seed=23):
    """O5 sample of a 3D output: n_lines random (x, y)
    lines with per_line random z each (>= 512 random outputs; outputs that
    share (x, y) share the oracle's pass over the x-y plane), plus every
    corner / edge / center point -- each axis at its extremes and its origin
    (0, m-1 for complex axes; -(m-1), 0, m-1 for centered ones) with z at
    0, 1, m-1."""
    rs = np.random.default_rng(seed)
    nx, ny, nz = shape
    i = rs.integers(0, nx, n_lines)
    j = rs.integers(0, ny, n_lines)
    rand = [np.ravel_multi_index((np.full(per_line, a), np.full(per_line, b),
                                  rs.choice(nz, per_line, replace=False)), shape) for a, b in zip(i, j)]
    def ext(n, c):
        return [0, (n - 1) // 2, n - 1] if c else [0, n - 1]
    edge = [np.ravel_multi_index((a, b, c), shape) for a in ext(nx, centered) for b in ext(ny, centered)
            for c in sorted({0, min(1, nz - 1), nz - 1})]
    return np.unique(np.concatenate(rand + [np.asarray(edge)]).astype(np.int64))


def test_config5a_cconv3d_512(idc):
    """C5a at full size (512^3, scaled 1/(1+|k|^2)) in the bench's launch
    configuration; >= 512 sampled outputs + corners/edges vs direct sums."""
    m = 512
    f, g = synthgen.cconv3d_inputs(m, m, m)
    F, G = dev(f), dev(g)
    idc.cconv3d(F, G)
    idx = c5_sample(f.shape, centered=False)
    assert idx.size >= 512 + 8
    oracle.set_work_cap(1e12)
    out = F.cpu().numpy().reshape(-1)[idx]
    del F, G
    torch.cuda.empty_cache()
    assert rel_l2(out, direct.cconv3d_at_large(f, g, idx)) < TOL


def test_config5b_hconv3d_512(idc):
    """C5b at full size ((2*512-1)^2 x 512 Hermitian, scaled); >= 512 sampled
    outputs + corners/edges vs direct sums (O5, Dot2-compensated)."""
    m = 512
    f, g = synthgen.hconv3d_inputs(m, m, m)
    F, G = dev(f), dev(g)
    idc.hconv3d(F, G)
    idx = c5_sample(f.shape, centered=True)
    assert idx.size >= 512 + 18
    oracle.set_work_cap(1e13)
    out = F.cpu().numpy().reshape(-1)[idx]
    del F, G
    torch.cuda.empty_cache()
    assert rel_l2(out, direct.hconv3d_at_lines(f, g, idx)) < TOL


# ------------------------------- 3D on the TMA pencils, element by element --
# Every axis of 64..4096 points runs the TMA pencil kernels (K5/K6 complex,
# K7/K8 centered) and 512-point z rows run the config-5 row kernels (K2/K3);
# these sizes reach each of them on x, y and z, element by element against
# the oracle's naive-DFT explicitly padded convolution (O2).

@pytest.mark.parametrize("shape", [(64, 64, 64), (128, 64, 64), (64, 128, 32), (512, 8, 8), (8, 512, 8),
                                   (8, 8, 512), (256, 64, 8), (128, 128, 128)])
def test_cconv3d_tma_vs_explicit(idc, shape):
    f, g = synthgen.cconv3d_inputs(*shape)
    ref = explicit.cconv3d(f, g)
    F, G = dev(f), dev(g)
    idc.cconv3d(F, G)
    assert rel_l2(F.cpu().numpy(), ref) < TOL


@pytest.mark.parametrize("ms", [(64, 64, 32), (32, 64, 64), (512, 4, 4), (4, 512, 4), (4, 4, 512), (64, 64, 16),
                                (128, 64, 8), (64, 64, 64), (128, 128, 64), (128, 128, 128)])
def test_hconv3d_tma_vs_explicit(idc, ms):
    f, g = synthgen.hconv3d_inputs(*ms)
    ref = explicit.hconv3d(f, g)
    F, G = dev(f), dev(g)
    idc.hconv3d(F, G)
    out = F.cpu().numpy()
    assert rel_l2(out, ref) < TOL
    p = out[:, :, 0]                          # kz = 0 plane stays Hermitian
    assert np.max(np.abs(p - np.conj(p[::-1, ::-1]))) < 1e-13 * np.max(np.abs(out))


# ------------------------------------------------ tall pencils (m >= 1024) --
# x axes of 1024-4096 points run the pencil kernels with 1-4-column tiles
# whose outputs leave by TMA tensor stores; a few columns (fewer than a
# tile: clipped stores) and batches (3D tensor maps) element by element.

@pytest.mark.parametrize("mx,my,B", [(2048, 1, 1), (2048, 2, 2), (4096, 2, 1), (4096, 8, 1), (1024, 2, 3)])
def test_cconv2d_tall(idc, mx, my, B):
    f, g = synthgen.cconv2d_inputs(mx, my, B)
    ref = np.stack([direct.cconv2d(f[b], g[b]) for b in range(B)])
    F, G = dev(f), dev(g)
    idc.cconv2d(F, G)
    assert rel_l2(F.cpu().numpy(), ref) < TOL


@pytest.mark.parametrize("mx,my", [(1024, 1), (1024, 2), (2048, 1), (2048, 4), (4096, 2)])
def test_hconv2d_tall(idc, mx, my):
    f, g = synthgen.hconv2d_inputs(mx, my)
    ref = direct.hconv2d(f, g)
    F, G = dev(f), dev(g)
    idc.hconv2d(F, G)
    assert rel_l2(F.cpu().numpy(), ref) < TOL


@pytest.mark.parametrize("mx,my", [(2048, 2), (1024, 4), (512, 1)])
def test_tconv2d_tall(idc, mx, my):
    from oracle import ternary2d
    arrs = []
    for r in range(3):
        a = synthgen.hconv2d_inputs(mx, my, roles=(r,))[0]
        arrs.append(np.concatenate([np.zeros((1, my), dtype=np.complex128), a], axis=0))
    ref = ternary2d.direct(*arrs)
    F, G, H = (dev(a) for a in arrs)
    idc.tconv2d(F, G, H)
    assert rel_l2(F.cpu().numpy(), ref) < TOL
