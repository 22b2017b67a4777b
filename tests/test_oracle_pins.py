"""Pins for the oracle: each oracle layer is checked against
something other than itself -- the paper's exact test families (P:272-280,
P:586-590), closed forms derived from the definitions, library routines
(numpy.convolve, scipy.signal.convolve), brute force on tiny inputs, and the
agreement of the three independent layers (direct / explicit DFT / implicit
equations).  CPU only."""
import itertools
import json
import os

import numpy as np
import pytest
import scipy.signal

import oracle
import synthgen
from oracle import closed, direct, explicit, implicit, rel_l2

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))
TOL = 1e-13


def crand(rng, *shape):
    return rng.uniform(-1, 1, shape) + 1j * rng.uniform(-1, 1, shape)


# ------------------------------------------------------------- generator --

def test_generator_golden_values():
    """Survey-recorded generator values (SURVEY §8(c) c.2 golden table), scalar and vector paths."""
    table = [
        (0, 0, -0.8937744387717883, -0.2190014850702946),
        (0, 1, -0.66175270967963873, 0.26315907116711035),
        (0, 1023, 0.98065952003095402, -0.36268712658876878),
        (1, 0, 0.21648158743906309, 0.40228377391156034),
        (2, 0, -0.84006212952359416, -0.43311435742256665),
        (4, 0, -0.37032426724444178, -0.22351060534859579),
        (5, 4095, 0.44745570744473584, -0.41578195556571407),
    ]
    for aid, idx, re, im in table:
        v = synthgen.uniform_at(aid, idx)
        assert v == complex(re, im)
        assert synthgen.uniform_complex(idx + 1, aid)[idx] == v


def test_generator_hermitian_recipes():
    f, = synthgen.hconv2d_inputs(4, 3, roles=(0,))
    c = 3
    for kx in range(1, 4):
        assert f[c - kx, 0] == np.conj(f[c + kx, 0])
    assert f[c, 0].imag == 0
    a, = synthgen.hconv3d_inputs(3, 2, 3, roles=(0,))
    nx, ny = a.shape[:2]
    for i, j in itertools.product(range(nx), range(ny)):
        assert a[i, j, 0] == np.conj(a[nx - 1 - i, ny - 1 - j, 0])


# ------------------------------------------------------------ D1 cconv1d --

@pytest.mark.parametrize("m", [1, 2, 8, 64, 1024])
def test_d1_paper_family(m):
    F = complex(*GOLD["cconv1d_family"]["F"])
    G = complex(*GOLD["cconv1d_family"]["G"])
    assert F == np.sqrt(3) + 1j * np.sqrt(7)
    f, g = closed.cconv1d_inputs(m, F, G)
    H = F * G * (np.arange(m) + 1) * np.exp(1j * np.arange(m))
    assert rel_l2(direct.cconv1d(f, g), H) < 1e-15
    assert rel_l2(closed.cconv1d(m), H) == 0


@pytest.mark.parametrize("m", [1, 3, 16, 100, 257])
def test_d1_numpy_convolve(rng, m):
    f, g = crand(rng, m), crand(rng, m)
    ref = np.convolve(f, g)[:m]          # textbook linear convolution, first m terms
    assert rel_l2(direct.cconv1d(f, g), ref) < TOL


def test_d1_special_cases(rng):
    m = 16
    g = crand(rng, m)
    for s in (0, 3, 15):
        f = np.zeros(m, complex)
        f[s] = 1
        ref = np.zeros(m, complex)
        ref[s:] = g[:m - s]
        assert np.array_equal(direct.cconv1d(f, g), ref)
    top = np.zeros(m, complex)
    top[m - 1] = 1
    assert np.array_equal(direct.cconv1d(top, top), np.zeros(m))       # no alias onto k = m-2
    ones = np.ones(m, complex)
    assert np.array_equal(direct.cconv1d(ones, ones), np.arange(1, m + 1).astype(complex))
    c = GOLD["cconv_m1"]
    assert direct.cconv1d(np.array([complex(*c["f"])]), np.array([complex(*c["g"])]))[0] == complex(*c["h"])


def test_d1_batch_independent(rng):
    f, g = crand(rng, 5, 32), crand(rng, 5, 32)
    h = direct.cconv1d(f, g)
    for b in range(5):
        assert np.array_equal(h[b], direct.cconv1d(f[b], g[b]))


# ------------------------------------------------------------ D2 hconv1d --

def ext1d(U):
    """[conj U_{m-1} .. conj U_1, Re U_0, U_1 .. U_{m-1}] (test-local, AMB-7)."""
    U = U.copy()
    U[0] = U[0].real
    return np.concatenate([np.conj(U[:0:-1]), U])


@pytest.mark.parametrize("m", [1, 2, 8, 512, 4096])
def test_d2_paper_family(m):
    F, G = GOLD["hconv1d_family"]["F"], GOLD["hconv1d_family"]["G"]
    k = np.arange(m)
    f, g = F * np.exp(1j * k), G * np.exp(1j * k)
    H = F * G * (2 * m - 1 - k) * np.exp(1j * k)
    assert rel_l2(direct.hconv1d(f, g), H) < 1e-15


@pytest.mark.parametrize("m", [1, 2, 6, 64, 255])
def test_d2_numpy_convolve(rng, m):
    f, g = crand(rng, m), crand(rng, m)
    full = np.convolve(ext1d(f), ext1d(g))             # indices -(2m-2)..(2m-2)
    ref = full[2 * (m - 1): 3 * (m - 1) + 1]
    assert rel_l2(direct.hconv1d(f, g), ref) < TOL


def test_d2_special_cases(rng):
    m = 12
    ones = np.ones(m, complex)
    assert np.array_equal(direct.hconv1d(ones, ones), (2 * m - 1 - np.arange(m)).astype(complex))
    top = np.zeros(m, complex)
    top[m - 1] = 1
    ref = np.zeros(m, complex)
    ref[0] = 2
    assert np.array_equal(direct.hconv1d(top, top), ref)
    # delta at s>0: h_k = g_{k-s} + g_{k+s} (conjugate extension, range-limited)
    g = crand(rng, m)
    s = 3
    d = np.zeros(m, complex)
    d[s] = 1
    G = ext1d(g)
    ref = np.array([(G[k - s + m - 1] if abs(k - s) <= m - 1 else 0) + (G[k + s + m - 1] if k + s <= m - 1 else 0)
                    for k in range(m)])
    assert rel_l2(direct.hconv1d(d, g), ref) < 1e-16
    c = GOLD["hconv_c1_dc"]
    h = direct.hconv1d(np.array([c["a"], 0j]), np.array([c["b"], 0j]))
    assert np.array_equal(h, np.array([c["a"] * c["b"], 0]))
    # projection (AMB-7): Im f_0 is discarded
    f = crand(rng, m)
    f2 = f.copy()
    f2[0] = f2[0].real
    assert np.array_equal(direct.hconv1d(f, g), direct.hconv1d(f2, g))


# ------------------------------------------------------------ D3 tconv1d --

@pytest.mark.parametrize("m", [1, 2, 3, 5, 8])
def test_d3_count_formula_vs_enumeration(m):
    rng_k = range(-(m - 1), m)
    for k in range(m):
        cnt = sum(1 for p in rng_k for q in rng_k if abs(k - p - q) <= m - 1)
        assert closed.ternary_count(m, k) == cnt
    if m == 8:
        assert closed.ternary_count(8, 0) == 169 and closed.ternary_count(8, 7) == 120


def test_d3_count_large():
    assert closed.ternary_count(4096, 0) == 3 * 4096 ** 2 - 3 * 4096 + 1 == 50319361
    assert closed.ternary_count(4096, 4095) == 33550336


@pytest.mark.parametrize("m", [2, 8, 64, 512])
def test_d3_closed_family(m):
    k = np.arange(m)
    e = np.exp(1j * k)
    F, G, H = np.sqrt(3), np.sqrt(5), np.sqrt(2)
    t = direct.tconv1d(F * e, G * e, H * e)
    assert rel_l2(t, closed.tconv1d(m, F, G, H)) < 1e-15


@pytest.mark.parametrize("m", [1, 2, 3, 7, 12])
def test_d3_brute_equals_two_stage(rng, m):
    f, g, h = crand(rng, m), crand(rng, m), crand(rng, m)
    assert rel_l2(direct.tconv1d(f, g, h), direct.tconv1d_brute(f, g, h)) < 1e-15


@pytest.mark.parametrize("m", [1, 4, 33, 128])
def test_d3_numpy_convolve(rng, m):
    f, g, h = crand(rng, m), crand(rng, m), crand(rng, m)
    full = np.convolve(np.convolve(ext1d(f), ext1d(g)), ext1d(h))   # -(3m-3)..(3m-3)
    ref = full[3 * (m - 1): 4 * (m - 1) + 1]
    assert rel_l2(direct.tconv1d(f, g, h), ref) < TOL


def test_d3_special_cases():
    c = GOLD["tconv_dc"]
    m = c["m"]
    a, b, cc = (np.zeros(m, complex) for _ in range(3))
    a[0], b[0], cc[0] = c["a"], c["b"], c["c"]
    ref = np.zeros(m, complex)
    ref[0] = c["a"] * c["b"] * c["c"]
    assert np.array_equal(direct.tconv1d(a, b, cc), ref)
    top = np.zeros(m, complex)
    top[m - 1] = 1
    ref = np.zeros(m, complex)
    ref[m - 1] = 3          # (m-1)+(m-1)-(m-1) in 3 orders; aliasing would need N < 4m-3
    assert np.array_equal(direct.tconv1d(top, top, top), ref)


# -------------------------------------------------------- D4/D6 complex ND --

@pytest.mark.parametrize("shape", [(1, 1), (4, 6), (8, 8), (3, 4, 4), (5, 3, 6)])
def test_d4_d6_closed_family(shape):
    f, g, H = closed.cconv_nd(shape)
    h = direct.cconv2d(f, g) if len(shape) == 2 else direct.cconv3d(f, g)
    assert rel_l2(h, H) < 1e-15


@pytest.mark.parametrize("shape", [(4, 6), (9, 5), (3, 4, 4), (4, 2, 5)])
def test_d4_d6_scipy_convolve(rng, shape):
    f, g = crand(rng, *shape), crand(rng, *shape)
    ref = scipy.signal.convolve(f, g, method="direct")[tuple(slice(0, n) for n in shape)]
    h = direct.cconv2d(f, g) if len(shape) == 2 else direct.cconv3d(f, g)
    assert rel_l2(h, ref) < TOL


def test_d4_separable(rng):
    a, b, c, d = crand(rng, 7), crand(rng, 5), crand(rng, 7), crand(rng, 5)
    h = direct.cconv2d(np.outer(a, b), np.outer(c, d))
    assert rel_l2(h, np.outer(direct.cconv1d(a, c), direct.cconv1d(b, d))) < TOL


# ------------------------------------------------------ D5/D7 Hermitian ND --

def test_d5_d7_closed_family():
    for ms in [(2, 2), (4, 3), (5, 6), (2, 2, 2), (3, 2, 4)]:
        f, g, H = closed.hconv_nd(ms)
        h = direct.hconv2d(f, g) if len(ms) == 2 else direct.hconv3d(f, g)
        assert rel_l2(h, H) < 1e-15, ms


def full2d_symmetric(rng, mx, my):
    """Random full centered (2mx-1, 2my-1) array with X_{-k} = conj X_k."""
    X = crand(rng, 2 * mx - 1, 2 * my - 1)
    X = 0.5 * (X + np.conj(X[::-1, ::-1]))
    return X


@pytest.mark.parametrize("mx,my", [(2, 2), (3, 4), (5, 3)])
def test_d5_scipy_convolve(rng, mx, my):
    X, Y = full2d_symmetric(rng, mx, my), full2d_symmetric(rng, mx, my)
    full = scipy.signal.convolve(X, Y, method="direct")        # centers at (2mx-2, 2my-2)
    ref = full[mx - 1: 3 * mx - 2, 2 * my - 2: 3 * my - 2]     # kx centered, ky = 0..my-1
    f, g = X[:, my - 1:], Y[:, my - 1:]
    assert rel_l2(direct.hconv2d(f, g), ref) < TOL


@pytest.mark.parametrize("ms", [(2, 2, 2), (3, 2, 3)])
def test_d7_scipy_convolve(rng, ms):
    mx, my, mz = ms
    X = crand(rng, 2 * mx - 1, 2 * my - 1, 2 * mz - 1)
    X = 0.5 * (X + np.conj(X[::-1, ::-1, ::-1]))
    Y = crand(rng, 2 * mx - 1, 2 * my - 1, 2 * mz - 1)
    Y = 0.5 * (Y + np.conj(Y[::-1, ::-1, ::-1]))
    full = scipy.signal.convolve(X, Y, method="direct")
    ref = full[mx - 1: 3 * mx - 2, my - 1: 3 * my - 2, 2 * mz - 2: 3 * mz - 2]
    assert rel_l2(direct.hconv3d(X[:, :, mz - 1:], Y[:, :, mz - 1:]), ref) < TOL


def test_d5_projection_and_output_symmetry(rng):
    """AMB-7: the ky=0 line is projected; the output ky=0 line is Hermitian."""
    mx, my = 4, 3
    f, g = crand(rng, 2 * mx - 1, my), crand(rng, 2 * mx - 1, my)
    fs = f.copy()
    fs[:, 0] = 0.5 * (f[:, 0] + np.conj(f[::-1, 0]))
    gs = g.copy()
    gs[:, 0] = 0.5 * (g[:, 0] + np.conj(g[::-1, 0]))
    h = direct.hconv2d(f, g)
    assert rel_l2(h, direct.hconv2d(fs, gs)) < 1e-15
    assert np.max(np.abs(h[:, 0] - np.conj(h[::-1, 0]))) < 1e-13 * np.max(np.abs(h))


# ------------------------------------------- O2 explicit vs O1 direct --

def test_explicit_matches_direct(rng):
    for m in (1, 2, 5, 16, 64):
        f, g, h = crand(rng, 2, m), crand(rng, 2, m), crand(rng, 2, m)
        assert rel_l2(explicit.cconv1d(f, g), direct.cconv1d(f, g)) < TOL
        assert rel_l2(explicit.hconv1d(f, g), direct.hconv1d(f, g)) < TOL
        assert rel_l2(explicit.tconv1d(f, g, h), direct.tconv1d(f, g, h)) < TOL
    for shp in [(4, 6), (8, 8)]:
        f, g = crand(rng, *shp), crand(rng, *shp)
        assert rel_l2(explicit.cconv2d(f, g), direct.cconv2d(f, g)) < TOL
    f, g = crand(rng, 3, 4, 5), crand(rng, 3, 4, 5)
    assert rel_l2(explicit.cconv3d(f, g), direct.cconv3d(f, g)) < TOL
    f, g = crand(rng, 7, 6), crand(rng, 7, 6)
    assert rel_l2(explicit.hconv2d(f, g), direct.hconv2d(f, g)) < TOL
    f, g = crand(rng, 5, 5, 4), crand(rng, 5, 5, 4)
    assert rel_l2(explicit.hconv3d(f, g), direct.hconv3d(f, g)) < TOL


def test_explicit_paper_families():
    for m in (8, 256, 1024):
        f, g = closed.cconv1d_inputs(m)
        assert rel_l2(explicit.cconv1d(f, g), closed.cconv1d(m)) < 1e-14
        k = np.arange(m)
        assert rel_l2(explicit.hconv1d(np.sqrt(3) * np.exp(1j * k), np.sqrt(5) * np.exp(1j * k)),
                      closed.hconv1d(m)) < 1e-14


# --------------------------------------- O3 implicit equations vs others --

def test_fftpad_spec_examples():
    for case in GOLD["fftpad_m2"]["cases"]:
        f = np.array([complex(*z) for z in case["f"]])
        e, o = implicit.fftpad_backward(f)
        assert np.allclose(e, [complex(*z) for z in case["even"]], atol=1e-15)
        assert np.allclose(o, [complex(*z) for z in case["odd"]], atol=1e-15)


def test_fft0pad_spec_delta():
    f = np.array([complex(*z) for z in GOLD["fft0pad_m2_delta"]["f"]])
    s = implicit.fft0pad_backward(f)
    for r in (-1, 0, 1):
        assert np.allclose(s[r], 1.0, atol=1e-15)
    assert np.allclose(implicit.fft0pad_forward(s, 2), f, atol=1e-15)


def test_padded_transforms_vs_naive_dft(rng):
    """Residue streams equal the naive N-point DFT of the explicitly padded vector."""
    m = 8
    U = crand(rng, m)
    N = 2 * m
    u = oracle.dft_matrix(N, range(N), range(m), +1) @ U
    e, o = implicit.fftpad_backward(U)
    assert rel_l2(e, u[0::2]) < 1e-14 and rel_l2(o, u[1::2]) < 1e-14
    A = crand(rng, 2 * m - 1)                       # centered, origin m-1
    N = 3 * m
    u = oracle.dft_matrix(N, range(N), np.arange(-(m - 1), m), +1) @ A
    s = implicit.fft0pad_backward(A)
    for r in (-1, 0, 1):
        assert rel_l2(s[r], u[(3 * np.arange(m) + r) % N]) < 1e-14
    B = crand(rng, 2 * m)
    B[0] = 0                                         # signed centered, origin m, U_{-m} = 0
    N = 4 * m
    u = oracle.dft_matrix(N, range(N), np.arange(-m, m), +1) @ B
    s = implicit.fft0tpad_backward(B)
    for r in (0, 1):
        assert rel_l2(s[r], u[2 * np.arange(2 * m) + r]) < 1e-14


@pytest.mark.parametrize("m", [2, 4, 16, 64])
def test_round_trips(rng, m):
    """"Returns the inverse"."""
    tol = 1e-13 * np.log2(max(m, 2))
    U = crand(rng, m)
    assert rel_l2(implicit.fftpad_forward(*implicit.fftpad_backward(U)), U) < tol
    A = crand(rng, 2 * m - 1)
    assert rel_l2(implicit.fft0pad_forward(implicit.fft0pad_backward(A), m), A) < tol
    B = crand(rng, 2 * m)
    B[0] = 0
    assert rel_l2(implicit.fft0tpad_forward(implicit.fft0tpad_backward(B), m), B[1:]) < tol


def test_implicit_matches_direct(rng):
    for m in (1, 2, 4, 16, 64):
        f, g = crand(rng, 3, m), crand(rng, 3, m)
        assert rel_l2(implicit.cconv1d(f, g), direct.cconv1d(f, g)) < TOL
    for m in (2, 4, 8, 32, 128):
        f, g, h = crand(rng, 3, m), crand(rng, 3, m), crand(rng, 3, m)
        assert rel_l2(implicit.hconv1d(f, g), direct.hconv1d(f, g)) < TOL
        assert rel_l2(implicit.tconv1d(f, g, h), direct.tconv1d(f, g, h)) < TOL
    f, g = crand(rng, 4, 6), crand(rng, 4, 6)
    assert rel_l2(implicit.cconv2d(f, g), direct.cconv2d(f, g)) < TOL
    f, g = crand(rng, 3, 4, 4), crand(rng, 3, 4, 4)
    assert rel_l2(implicit.cconv3d(f, g), direct.cconv3d(f, g)) < TOL
    f, g = crand(rng, 7, 6), crand(rng, 7, 6)
    assert rel_l2(implicit.hconv2d(f, g), direct.hconv2d(f, g)) < TOL
    f, g = crand(rng, 5, 5, 4), crand(rng, 5, 5, 4)
    assert rel_l2(implicit.hconv3d(f, g), direct.hconv3d(f, g)) < TOL


def test_implicit_paper_families():
    for m in (4, 64, 1024):
        f, g = closed.cconv1d_inputs(m)
        assert rel_l2(implicit.cconv1d(f, g), closed.cconv1d(m)) < 1e-14
        k = np.arange(m)
        assert rel_l2(implicit.hconv1d(np.sqrt(3) * np.exp(1j * k), np.sqrt(5) * np.exp(1j * k)),
                      closed.hconv1d(m)) < 1e-14


def test_hermitian_w_symmetry(rng):
    """w_{k,r} = conj(w_{m-k,r})."""
    m = 8
    U = crand(rng, m)
    for r in (-1, 0, 1):
        w = implicit.hermitian_w(U, r)
        for k in range(1, m):
            assert abs(w[k] - np.conj(w[m - k])) < 1e-15


def test_linearity_and_symmetry(rng):
    m = 32
    f1, f2, g = crand(rng, m), crand(rng, m), crand(rng, m)
    a, b = 0.3 - 1.2j, 2.0 + 0.5j
    lhs = direct.cconv1d(a * f1 + b * f2, g)
    rhs = a * direct.cconv1d(f1, g) + b * direct.cconv1d(f2, g)
    assert rel_l2(lhs, rhs) < 1e-14
    assert rel_l2(direct.cconv1d(f1, g), direct.cconv1d(g, f1)) < 1e-15
    d = np.zeros(m, complex)
    d[0] = 1
    assert np.array_equal(direct.cconv1d(d, g), g)


# ------------------------------------------------------- memory formulas --

def test_memory_formulas():
    mw = GOLD["memory_words"]
    assert oracle.memory.cconv2d_implicit(1024, 1024) == mw["cconv2d_1024x1024"]
    assert oracle.memory.hconv2d_implicit(4, 4) == mw["hconv2d_4x4"] == 6 * 16 + 4 + 2
    assert oracle.memory.cconv3d_implicit(1, 1, 1) == mw["cconv3d_1x1x1"]
    assert oracle.memory.hconv2d_implicit(2048, 2048) == mw["hconv2d_2048x2048"] == 6 * 2048 ** 2 + 2048 + 2
    assert oracle.memory.cconv3d_implicit(512, 512, 512) == mw["cconv3d_512x512x512"]
    m = 512
    # P:894 is internally inconsistent: its itemised left side
    # 6mx(2my-1)mz + 2(my+1)mz + 2(mz/2+1) exceeds its closed right side
    # 12mxmymz - 6mxmz + 2mymz + mz + 2 by exactly 2mz (reading AMB-21).
    rhs = 12 * m ** 3 - 6 * m * m + 2 * m * m + m + 2
    assert rhs == mw["hconv3d_512x512x512"]
    assert oracle.memory.hconv3d_implicit(m, m, m) - rhs == 2 * m


def test_large_sampled_oracles_agree(rng):
    """The mirror-on-the-fly / parallel sampled routines equal the plain ones."""
    f, g = synthgen.hconv3d_inputs(4, 3, 5)
    idx = np.arange(f.size)
    assert rel_l2(direct.hconv3d_at_large(f, g, idx), direct.hconv3d_at(f, g, idx)) < 1e-15
    a, b = crand(rng, 5, 4, 6), crand(rng, 5, 4, 6)
    idx = np.arange(a.size)
    assert rel_l2(direct.cconv3d_at_large(a, b, idx), direct.cconv_nd_at(a, b, idx)) < 1e-15


@pytest.mark.parametrize("ms", [(1, 1, 1), (4, 3, 5), (2, 5, 9), (3, 2, 1), (5, 6, 7), (2, 2, 16)])
def test_hconv3d_at_lines_equals_plain(ms):
    """The z-run / Dot2 sampled D7 (O5 for config 5b) sums the same terms as
    the plain extended-array loop: agreement to rounding at every output."""
    f, g = synthgen.hconv3d_inputs(*ms)
    idx = np.arange(f.size)
    assert rel_l2(direct.hconv3d_at_lines(f, g, idx), direct.hconv3d_at(f, g, idx)) < 1e-15


def test_hconv3d_at_lines_closed_family_and_scipy(rng):
    """Pinned against the closed form (2mx-1-|kx|)(2my-1-|ky|)(2mz-1-kz) FG
    e^{i(kx+ky+kz)} and against scipy's direct convolution of the extended
    arrays, independently of the plain loop."""
    f, g, H = closed.hconv_nd((6, 5, 12))
    idx = np.arange(f.size)
    assert rel_l2(direct.hconv3d_at_lines(f, g, idx), H.reshape(-1)) < 1e-15
    mx, my, mz = 3, 2, 5
    X = crand(rng, 2 * mx - 1, 2 * my - 1, 2 * mz - 1)
    X = 0.5 * (X + np.conj(X[::-1, ::-1, ::-1]))
    Y = crand(rng, 2 * mx - 1, 2 * my - 1, 2 * mz - 1)
    Y = 0.5 * (Y + np.conj(Y[::-1, ::-1, ::-1]))
    ref = scipy.signal.convolve(X, Y, method="direct")[mx - 1: 3 * mx - 2, my - 1: 3 * my - 2, 2 * mz - 2: 3 * mz - 2]
    a, b = X[:, :, mz - 1:].copy(), Y[:, :, mz - 1:].copy()
    idx = np.arange(a.size)
    assert rel_l2(direct.hconv3d_at_lines(a, b, idx), ref.reshape(-1)) < 1e-14


def test_fast_generator_bitwise():
    for aid, start, n in [(0, 0, 1000), (9, 77, 5000)]:
        assert np.array_equal(synthgen.uniform_complex_fast(n, aid, start=start),
                              synthgen.uniform_complex(n, aid, start=start))
