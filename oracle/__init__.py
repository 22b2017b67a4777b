"""Oracle for the implicitly dealiased convolutions -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with the CUDA path (``paper_1008_1366_b200``) and never imports
it; the only module both sides use is ``synthgen`` (seeded inputs, no method
arithmetic).

Citations: "P:<line>" = /root/reference/PAPER.md (Bowman & Roberts, "Efficient
Dealiased Convolutions without Padding", arXiv 1008.1366), "S:<line>" =
SPEC.md, AMB-n = the readings listed in DESIGN.md / SURVEY.md §8(c) c.3.

Layers:

* O1 ``direct.*``  -- direct sums D1-D7 in C (oracle/direct.c), TwoProd +
  Neumaier compensated accumulation, OpenMP.  The definition written out.
* O2 ``explicit.*`` -- naive-DFT explicitly zero-padded convolution: pad each
  axis to N = 2m / 3m / 4m, dense DFT
  matrices with exact integer angle reduction and long-double trig, pointwise
  product, inverse DFT, 1/N, extract the dealiased range (AMB-6).
* O3 ``implicit.*`` -- the paper's residue-stream equations evaluated with
  naive DFTs, step by step in the paper's notation: Eqs. cconv1backward /
  cconv1forward, fft0backwardA/B + fft0forward, the
  Hermitian w_{k,r} + fft0forwardB, the ternary backward/forward
  (P:1015-1027), fft0tbackward/forward; the 2D/3D compositions
  cconv2, conv2, cconv3, Hermitian 3D
  (AMB-9).
* O4 ``closed.*`` -- the paper's exact test families
  and their derived 2D/3D/ternary analogues.
* O1b ``ternary2d.*`` -- the 2D centered Hermitian ternary sum (Function
  tconv2, NEXT-2): two-stage direct 2D convolution and a brute-force loop.
* O5 ``application.*`` -- the 2D pseudospectral Euler sum of P:867-876
  written out (pinned by a two-mode closed form and by its decomposition into
  D5 direct sums).

Parity status: every function here is pinned by tests/test_oracle_*.py
against closed forms, library routines (numpy.convolve), brute force or the
agreement of independent layers; none is "parity unpinned" except where its
docstring says so.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _cpu_has(*flags) -> bool:
    try:
        with open("/proc/cpuinfo") as fh:
            have = set()
            for line in fh:
                if line.startswith("flags"):
                    have = set(line.split(":", 1)[1].split())
                    break
        return all(f in have for f in flags)
    except OSError:
        return False


def build(force: bool = False) -> str:
    """Compile oracle/direct.c into oracle/liboracle.so (gcc, OpenMP)."""
    so = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "direct.c")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        # hardware FMA keeps TwoProd exact and fast (a libm fma() call is
        # ~20x slower); -ffp-contract=off keeps the compiler from fusing the
        # error-free transforms themselves
        isa = "-mavx2 -mfma" if _cpu_has("avx2", "fma") else ""
        cmd = f"gcc -O3 {isa} -fopenmp -ffp-contract=off -fPIC -shared -o {so} {src} -lm"
        if os.system(cmd) != 0:
            raise RuntimeError("oracle build failed: " + cmd)
    return so


def lib():
    global _LIB
    if _LIB is None:
        _LIB = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I = ctypes.c_int64
        for name, args in {
            "orc_cconv1d": [P, P, P, I, I],
            "orc_hconv1d": [P, P, P, I, I],
            "orc_tconv1d": [P, P, P, P, I, I],
            "orc_tconv1d_brute": [P, P, P, P, I],
            "orc_cconv3d_at": [P, P, I, I, I, P, I, P],
            "orc_hconv3d_at": [P, P, I, I, I, P, I, P],
            "orc_hconv2d_at": [P, P, I, I, P, I, P],
            "orc_hconv3d_at_mirror": [P, P, I, I, I, P, I, P],
            "orc_cconv3d_at_par": [P, P, I, I, I, P, I, P],
            "orc_hconv3d_at_zlist": [P, P, I, I, I, I, I, P, I, P],
        }.items():
            fn = getattr(_LIB, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        _LIB.orc_set_work_cap.argtypes = [ctypes.c_double]
        _LIB.orc_set_work_cap.restype = None
    return _LIB


def set_work_cap(macs: float) -> None:
    lib().orc_set_work_cap(float(macs))


def _c(a):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc, what):
    if rc == -1:
        raise RuntimeError(f"{what}: work cap exceeded (oracle.set_work_cap)")
    if rc != 0:
        raise ValueError(f"{what}: bad arguments (rc={rc})")


# =========================================================== O1 direct sums ==

class direct:
    """O1: the definitions D1-D7 as direct sums in C."""

    @staticmethod
    def cconv1d(f, g):
        """D1: h_k = sum_{p=0}^k f_p g_{k-p}; f, g shape (..., m)."""
        f, g = _c(f), _c(g)
        m = f.shape[-1]
        B = f.size // m
        h = np.empty_like(f)
        _check(lib().orc_cconv1d(_ptr(f), _ptr(g), _ptr(h), m, B), "cconv1d")
        return h

    @staticmethod
    def hconv1d(f, g):
        """D2: centered Hermitian; f_{-p} = conj f_p, f_0 := Re f_0."""
        f, g = _c(f), _c(g)
        m = f.shape[-1]
        B = f.size // m
        h = np.empty_like(f)
        _check(lib().orc_hconv1d(_ptr(f), _ptr(g), _ptr(h), m, B), "hconv1d")
        return h

    @staticmethod
    def tconv1d(f, g, h):
        """D3 via the exact two-stage O(m^2) form."""
        f, g, h = _c(f), _c(g), _c(h)
        m = f.shape[-1]
        B = f.size // m
        t = np.empty_like(f)
        _check(lib().orc_tconv1d(_ptr(f), _ptr(g), _ptr(h), _ptr(t), m, B), "tconv1d")
        return t

    @staticmethod
    def tconv1d_brute(f, g, h):
        """D3 literal O(m^3) triple sum (one vector, small m)."""
        f, g, h = _c(f), _c(g), _c(h)
        m = f.shape[-1]
        t = np.empty_like(f)
        _check(lib().orc_tconv1d_brute(_ptr(f), _ptr(g), _ptr(h), _ptr(t), m), "tconv1d_brute")
        return t

    @staticmethod
    def cconv_nd_at(f, g, idx):
        """D4/D6 at the given linear output indices (f, g of shape (n0, n1[, n2]))."""
        f, g = _c(f), _c(g)
        shp = f.shape + (1,) * (3 - f.ndim)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.empty(idx.size, dtype=np.complex128)
        _check(lib().orc_cconv3d_at(_ptr(f), _ptr(g), shp[0], shp[1], shp[2], _ptr(idx), idx.size, _ptr(out)),
               "cconv_nd_at")
        return out

    @staticmethod
    def cconv2d(f, g):
        """D4, full output."""
        f = _c(f)
        return direct.cconv_nd_at(f, g, np.arange(f.size)).reshape(f.shape)

    @staticmethod
    def cconv3d(f, g):
        """D6, full output."""
        f = _c(f)
        return direct.cconv_nd_at(f, g, np.arange(f.size)).reshape(f.shape)

    @staticmethod
    def hconv2d_at(f, g, idx):
        """D5 at linear indices of the (2mx-1, my) storage."""
        f, g = _c(f), _c(g)
        mx = (f.shape[0] + 1) // 2
        my = f.shape[1]
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.empty(idx.size, dtype=np.complex128)
        _check(lib().orc_hconv2d_at(_ptr(f), _ptr(g), mx, my, _ptr(idx), idx.size, _ptr(out)), "hconv2d_at")
        return out

    @staticmethod
    def hconv2d(f, g):
        """D5, full output (2mx-1, my)."""
        f = _c(f)
        return direct.hconv2d_at(f, g, np.arange(f.size)).reshape(f.shape)

    @staticmethod
    def hconv3d_at(f, g, idx):
        """D7 at linear indices of the (2mx-1, 2my-1, mz) storage (AMB-9)."""
        f, g = _c(f), _c(g)
        mx = (f.shape[0] + 1) // 2
        my = (f.shape[1] + 1) // 2
        mz = f.shape[2]
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.empty(idx.size, dtype=np.complex128)
        _check(lib().orc_hconv3d_at(_ptr(f), _ptr(g), mx, my, mz, _ptr(idx), idx.size, _ptr(out)), "hconv3d_at")
        return out

    @staticmethod
    def hconv3d_at_large(f, g, idx):
        """D7 at sampled outputs of a large array: mirror/projection on the fly
        (no 8x extended copy), each point parallelised over px."""
        f, g = _c(f), _c(g)
        mx, my, mz = (f.shape[0] + 1) // 2, (f.shape[1] + 1) // 2, f.shape[2]
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.empty(idx.size, dtype=np.complex128)
        _check(lib().orc_hconv3d_at_mirror(_ptr(f), _ptr(g), mx, my, mz, _ptr(idx), idx.size, _ptr(out)),
               "hconv3d_at_large")
        return out

    @staticmethod
    def hconv3d_at_lines(f, g, idx):
        """D7 at sampled outputs of a large array (O5 for config 5b): the same
        terms as hconv3d_at, read in place from the stored half-space (mirror
        and kz = 0 projection resolved per z run, AMB-7) and summed as Dot2
        compensated dot products; outputs sharing (kx, ky) share one pass
        over the x-y plane (oracle/direct.c orc_hconv3d_at_zlist)."""
        f, g = _c(f), _c(g)
        mx, my, mz = (f.shape[0] + 1) // 2, (f.shape[1] + 1) // 2, f.shape[2]
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        i, j, l = np.unravel_index(idx, f.shape)
        out = np.empty(idx.size, dtype=np.complex128)
        for (a, b) in sorted(set(zip(i.tolist(), j.tolist()))):
            sel = np.nonzero((i == a) & (j == b))[0]
            kz = np.ascontiguousarray(l[sel], dtype=np.int64)
            res = np.empty(kz.size, dtype=np.complex128)
            _check(lib().orc_hconv3d_at_zlist(_ptr(f), _ptr(g), mx, my, mz, a - (mx - 1), b - (my - 1), _ptr(kz),
                                              kz.size, _ptr(res)), "hconv3d_at_lines")
            out[sel] = res
        return out

    @staticmethod
    def cconv3d_at_large(f, g, idx):
        """D6 at sampled outputs of a large array, each point parallelised."""
        f, g = _c(f), _c(g)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.empty(idx.size, dtype=np.complex128)
        _check(lib().orc_cconv3d_at_par(_ptr(f), _ptr(g), *f.shape, _ptr(idx), idx.size, _ptr(out)),
               "cconv3d_at_large")
        return out

    @staticmethod
    def hconv3d(f, g):
        """D7 full output."""
        f = _c(f)
        return direct.hconv3d_at(f, g, np.arange(f.size)).reshape(f.shape)


# ================================================== roots of unity (exact) ==

def zeta(N: int, k) -> np.ndarray:
    """zeta_N^k = exp(2 pi i k / N), with the integer argument
    reduced exactly mod N and cos/sin evaluated in long double."""
    k = np.asarray(k, dtype=np.int64) % N
    # 2*pi in long double via 8*atan(1) for the extra digits
    ang = np.longdouble(8) * np.arctan(np.longdouble(1)) * k.astype(np.longdouble) / np.longdouble(N)
    return (np.cos(ang).astype(np.float64) + 1j * np.sin(ang).astype(np.float64)).astype(np.complex128)


def dft_matrix(N: int, rows, cols, sign: int) -> np.ndarray:
    """Dense matrix W[j, k] = zeta_N^{sign * j * k} for j in rows, k in cols."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    return zeta(N, sign * np.outer(rows, cols))


def _apply_axis(M: np.ndarray, a: np.ndarray, axis: int) -> np.ndarray:
    """Contract matrix M[j, k] with a along `axis` (k), result index j in place."""
    a = np.moveaxis(a, axis, -1)
    out = a @ M.T
    return np.moveaxis(out, -1, axis)


# ================================================ O2 explicit padded DFTs ==

class explicit:
    """O2: naive-DFT explicitly zero-padded convolutions."""

    @staticmethod
    def cconv_nd(f, g, axes_m):
        """Complex axes: pad each axis of length m to N = 2m,
        backward DFT (sign +), product, forward DFT (sign -), /N,
        keep indices 0..m-1."""
        f, g = _c(f), _c(g)
        nd = len(axes_m)
        lead = f.ndim - nd
        F, G = f, g
        for ax, m in enumerate(axes_m):
            N = 2 * m
            W = dft_matrix(N, range(N), range(m), +1)
            F = _apply_axis(W, F, lead + ax)
            G = _apply_axis(W, G, lead + ax)
        P = F * G
        for ax, m in enumerate(axes_m):
            N = 2 * m
            W = dft_matrix(N, range(m), range(N), -1) / N
            P = _apply_axis(W, P, lead + ax)
        return P

    @staticmethod
    def cconv1d(f, g):
        f = _c(f)
        return explicit.cconv_nd(f, g, (f.shape[-1],))

    @staticmethod
    def cconv2d(f, g):
        f = _c(f)
        return explicit.cconv_nd(f, g, f.shape[-2:])

    @staticmethod
    def cconv3d(f, g):
        f = _c(f)
        return explicit.cconv_nd(f, g, f.shape[-3:])

    @staticmethod
    def _hermitian_full1d(U):
        """(..., m) half spectrum -> (..., 2m-1) centered full spectrum (AMB-7)."""
        U = _c(U).copy()
        U[..., 0] = U[..., 0].real
        return np.concatenate([np.conj(U[..., :0:-1]), U], axis=-1)

    @staticmethod
    def _centered_conv(full_arrays, ms, N_of_m, out_slices):
        """Generic explicit centered convolution of len(full_arrays) inputs.
        Each axis a holds centered indices k = -(m_a-1)..(m_a-1) at position
        k + (m_a-1); it is padded to N_a = N_of_m(m_a) with index k placed at
        k mod N_a (backward DFT over all N_a points), the inputs are
        multiplied, the forward DFT divided by N_a is evaluated at the output
        wavenumbers out_slices[a] (a list of signed k)."""
        prods = None
        for A in full_arrays:
            X = _c(A)
            for ax, m in enumerate(ms):
                N = N_of_m(m)
                ks = np.arange(-(m - 1), m)
                W = dft_matrix(N, range(N), ks, +1)
                X = _apply_axis(W, X, ax)
            prods = X if prods is None else prods * X
        P = prods
        for ax, m in enumerate(ms):
            N = N_of_m(m)
            W = dft_matrix(N, out_slices[ax], range(N), -1) / N
            P = _apply_axis(W, P, ax)
        return P

    @staticmethod
    def hconv1d(f, g):
        """Centered Hermitian, 2/3 rule with N = 3m."""
        f, g = _c(f), _c(g)
        m = f.shape[-1]
        F = explicit._hermitian_full1d(f)
        G = explicit._hermitian_full1d(g)
        N = 3 * m
        ks = np.arange(-(m - 1), m)
        Wb = dft_matrix(N, range(N), ks, +1)
        Wf = dft_matrix(N, range(m), range(N), -1) / N
        return (F @ Wb.T * (G @ Wb.T)) @ Wf.T

    @staticmethod
    def tconv1d(f, g, h):
        """Centered Hermitian ternary, N = 4m."""
        f, g, h = _c(f), _c(g), _c(h)
        m = f.shape[-1]
        N = 4 * m
        ks = np.arange(-(m - 1), m)
        Wb = dft_matrix(N, range(N), ks, +1)
        Wf = dft_matrix(N, range(m), range(N), -1) / N
        X = [explicit._hermitian_full1d(a) @ Wb.T for a in (f, g, h)]
        return (X[0] * X[1] * X[2]) @ Wf.T

    @staticmethod
    def _hermitian_full2d(A):
        """(2mx-1, my) -> (2mx-1, 2my-1) full centered array; ky=0 line
        projected (U + conj U(-kx))/2 (AMB-7)."""
        A = _c(A)
        nx, my = A.shape
        X = np.empty((nx, 2 * my - 1), dtype=np.complex128)
        X[:, my - 1:] = A
        X[:, my - 1] = 0.5 * (A[:, 0] + np.conj(A[::-1, 0]))
        # U_{kx,-ky} = conj(U_{-kx,ky})
        X[:, :my - 1] = np.conj(A[::-1, :0:-1])
        return X

    @staticmethod
    def hconv2d(f, g):
        """D5 explicitly padded, N = 3m on both axes, output kx centered, ky>=0."""
        nx, my = f.shape
        mx = (nx + 1) // 2
        F = explicit._hermitian_full2d(f)
        G = explicit._hermitian_full2d(g)
        out = explicit._centered_conv([F, G], (mx, my), lambda m: 3 * m,
                                      [np.arange(-(mx - 1), mx), np.arange(0, my)])
        return out

    @staticmethod
    def _hermitian_full3d(A):
        """(2mx-1, 2my-1, mz) -> (2mx-1, 2my-1, 2mz-1); kz=0 plane projected."""
        A = _c(A)
        nx, ny, mz = A.shape
        X = np.empty((nx, ny, 2 * mz - 1), dtype=np.complex128)
        X[:, :, mz - 1:] = A
        X[:, :, mz - 1] = 0.5 * (A[:, :, 0] + np.conj(A[::-1, ::-1, 0]))
        X[:, :, :mz - 1] = np.conj(A[::-1, ::-1, :0:-1])
        return X

    @staticmethod
    def hconv3d(f, g):
        nx, ny, mz = f.shape
        mx, my = (nx + 1) // 2, (ny + 1) // 2
        F = explicit._hermitian_full3d(f)
        G = explicit._hermitian_full3d(g)
        return explicit._centered_conv([F, G], (mx, my, mz), lambda m: 3 * m,
                                       [np.arange(-(mx - 1), mx), np.arange(-(my - 1), my), np.arange(0, mz)])


# ============================================ O3 implicit (paper equations) ==

def _dftm(m, sign):
    """size-m DFT matrix zeta_m^{sign l k} (rows l, cols k)."""
    return dft_matrix(m, range(m), range(m), sign)


class implicit:
    """O3: the paper's implicit-padding equations with naive size-m DFTs."""

    # ---- complex 1/2 rule, Eqs. cconv1backward / cconv1forward
    @staticmethod
    def fftpad_backward(U):
        """Returns (even, odd) residue streams u_{2l}, u_{2l+1}, l = 0..m-1:
        u_{2l} = sum_k zeta_m^{lk} U_k ; u_{2l+1} = sum_k zeta_m^{lk} zeta_{2m}^k U_k."""
        U = _c(U)
        m = U.shape[-1]
        Wm = _dftm(m, +1)
        tw = zeta(2 * m, np.arange(m))
        return U @ Wm.T, (U * tw) @ Wm.T

    @staticmethod
    def fftpad_forward(ue, uo):
        """2m U_k = sum_l zeta_m^{-kl} u_{2l} + zeta_{2m}^{-k} sum_l zeta_m^{-kl} u_{2l+1}; returns U (divided by 2m)."""
        m = ue.shape[-1]
        Wm = _dftm(m, -1)
        tw = zeta(2 * m, -np.arange(m))
        return (ue @ Wm.T + tw * (uo @ Wm.T)) / (2 * m)

    @staticmethod
    def cconv1d(f, g):
        """Function cconv: products of the residue streams."""
        fe, fo = implicit.fftpad_backward(f)
        ge, go = implicit.fftpad_backward(g)
        return implicit.fftpad_forward(fe * ge, fo * go)

    # ---- general p/q padding
    @staticmethod
    def fftpad_pq_backward(U, p, q):
        """pm modes U (..., pm) implicitly padded to qm: returns dict r -> stream
        u_{q l + r}, l < m, u_{ql+r} = sum_s zeta_m^{ls} sum_{t<p} zeta_{qm}^{r(tm+s)} U_{tm+s}."""
        U = _c(U)
        m = U.shape[-1] // p
        Wm = _dftm(m, +1)
        s = np.arange(m)
        out = {}
        for r in range(q):
            w = sum(zeta(q * m, r * (t * m + s)) * U[..., t * m:(t + 1) * m] for t in range(p))
            out[r] = w @ Wm.T
        return out

    @staticmethod
    def fftpad_pq_forward(streams, p, q, m):
        """qm U_k = sum_{r<q} zeta_{qm}^{-rk} sum_l zeta_m^{-kl} u_{ql+r}, k < pm; returns U."""
        k = np.arange(p * m)
        Wk = dft_matrix(m, k, range(m), -1)
        out = 0
        for r in range(q):
            out = out + zeta(q * m, -r * k) * (streams[r] @ Wk.T)
        return out / (q * m)

    @staticmethod
    def cconv1d_pq(f, g, p, q):
        """Complex convolution with p/q implicit padding: products of the q residue streams."""
        m = f.shape[-1] // p
        sf = implicit.fftpad_pq_backward(f, p, q)
        sg = implicit.fftpad_pq_backward(g, p, q)
        return implicit.fftpad_pq_forward({r: sf[r] * sg[r] for r in range(q)}, p, q, m)

    # ---- centered 2/3 rule, Eqs. fft0backwardA/B, fft0forward
    @staticmethod
    def fft0pad_backward(A):
        """A: (..., 2m-1) centered with origin at index m-1.  Returns dict
        r -> stream u_{3l+r}, l = 0..m-1, r in {-1, 0, 1}:
        w_{0,r} = U_0, w_{k,r} = zeta_{3m}^{rk}(U_k + zeta_3^{-r} U_{k-m})."""
        A = _c(A)
        m = (A.shape[-1] + 1) // 2
        Up = A[..., m - 1:]                       # U_k, k = 0..m-1
        Un = np.concatenate([np.zeros_like(A[..., :1]), A[..., :m - 1]], axis=-1)  # U_{k-m}, k=1..m-1 (k=0 unused)
        Wm = _dftm(m, +1)
        k = np.arange(m)
        streams = {}
        for r in (-1, 0, 1):
            w = zeta(3 * m, r * k) * (Up + zeta(3, -r) * Un)
            w[..., 0] = Up[..., 0]
            streams[r] = w @ Wm.T
        return streams

    @staticmethod
    def fft0pad_forward(streams, m):
        """3m U_k = sum_r zeta_{3m}^{-rk} sum_l zeta_m^{-lk} u_{3l+r}, k = -m+1..m-1."""
        ks = np.arange(-(m - 1), m)
        Wk = dft_matrix(m, ks, range(m), -1)
        out = 0
        for r in (-1, 0, 1):
            out = out + zeta(3 * m, -r * ks) * (streams[r] @ Wk.T)
        return out / (3 * m)

    # ---- centered Hermitian: w_{k,r} with conj(U_{m-k})
    @staticmethod
    def hermitian_w(U, r):
        """w_{0,r} = U_0 (projected real, AMB-7); w_{k,r} = zeta_{3m}^{rk}(U_k + zeta_3^{-r} conj(U_{m-k}))."""
        U = _c(U)
        m = U.shape[-1]
        k = np.arange(m)
        Umk = np.conj(np.concatenate([U[..., :1], U[..., :0:-1]], axis=-1))  # conj(U_{m-k}); k=0 unused
        w = zeta(3 * m, r * k) * (U + zeta(3, -r) * Umk)
        w[..., 0] = U[..., 0].real
        return w

    @staticmethod
    def crfft(W, n):
        """Complex-to-real backward transform of size n from the first n//2+1
        components (Hermitian extension W_{n-k} = conj W_k)."""
        c = n // 2
        half = W[..., :c + 1].copy()
        half[..., 0] = half[..., 0].real
        if n % 2 == 0:
            half[..., c] = half[..., c].real
        full = np.concatenate([half, np.conj(half[..., 1:n - c][..., ::-1])], axis=-1)
        u = full @ _dftm(n, +1).T
        return u.real

    @staticmethod
    def rcfft(u, n):
        """Real-to-complex forward transform: first n//2+1 frequencies."""
        return u.astype(np.complex128) @ dft_matrix(n, range(n // 2 + 1), range(n), -1).T

    @staticmethod
    def hconv1d(f, g):
        """Centered Hermitian convolution via three c2r of the first c+1 w_{k,r},
        real products, r2c + Hermitian symmetry, Eq. fft0forwardB."""
        f, g = _c(f), _c(g)
        m = f.shape[-1]
        c = m // 2
        k = np.arange(m)
        out = 0
        for r in (-1, 0, 1):
            uf = implicit.crfft(implicit.hermitian_w(f, r), m)
            ug = implicit.crfft(implicit.hermitian_w(g, r), m)
            P = implicit.rcfft(uf * ug, m)                       # k = 0..c
            Pfull = np.concatenate([P, np.conj(P[..., 1:m - c][..., ::-1])], axis=-1)  # k > c by symmetry
            out = out + zeta(3 * m, -r * k) * Pfull
        return out / (3 * m)

    # ---- Hermitian ternary, N = 4m, two residues of size 2m
    @staticmethod
    def tconv1d(f, g, h):
        """u_{2l+r} = c2r_{2m}{zeta_{4m}^{rk} U_k : k = 0..m} with U_m = 0;
        4m U_k = sum_r zeta_{4m}^{-rk} sum_l zeta_{2m}^{-lk} u_{2l+r}, k = 0..m-1."""
        f, g, h = _c(f), _c(g), _c(h)
        m = f.shape[-1]
        k = np.arange(m + 1)
        out = 0
        for r in (0, 1):
            prod = 1.0
            for U in (f, g, h):
                Uext = np.concatenate([U, np.zeros_like(U[..., :1])], axis=-1)  # U_m = 0
                Uext[..., 0] = Uext[..., 0].real
                prod = prod * implicit.crfft(zeta(4 * m, r * k) * Uext, 2 * m)
            P = implicit.rcfft(prod, 2 * m)[..., :m]
            out = out + zeta(4 * m, -r * np.arange(m)) * P
        return out / (4 * m)

    # ---- signed centered 4m transform, Eqs. fft0tbackward/forward
    @staticmethod
    def fft0tpad_backward(A):
        """A: (..., 2m) with A[0] = 0 (U_{-m}), origin at index m.  Returns the
        two streams u_{2l+r}, l = 0..2m-1, r = 0, 1 (first form of Eq. fft0tbackward)."""
        A = _c(A)
        m = A.shape[-1] // 2
        ks = np.arange(-m, m)
        W = dft_matrix(2 * m, range(2 * m), ks, +1)
        return {r: (zeta(4 * m, r * ks) * A) @ W.T for r in (0, 1)}

    @staticmethod
    def fft0tpad_forward(streams, m):
        """4m U_k = sum_r zeta_{4m}^{-rk} sum_l zeta_{2m}^{-lk} u_{2l+r}, k = -m+1..m-1 (first form)."""
        ks = np.arange(-(m - 1), m)
        Wk = dft_matrix(2 * m, ks, range(2 * m), -1)
        out = sum(zeta(4 * m, -r * ks) * (streams[r] @ Wk.T) for r in (0, 1))
        return out / (4 * m)

    # ---- 2D / 3D compositions
    @staticmethod
    def cconv2d(f, g):
        """Function cconv2: fftpadBackward on every column j, cconv on
        every row of both streams, fftpadForward on every column."""
        f, g = _c(f), _c(g)
        fT_e, fT_o = implicit.fftpad_backward(np.swapaxes(f, -1, -2))
        gT_e, gT_o = implicit.fftpad_backward(np.swapaxes(g, -1, -2))
        # rows of the x-residue streams: (..., l, y)
        re = implicit.cconv1d(np.swapaxes(fT_e, -1, -2), np.swapaxes(gT_e, -1, -2))
        ro = implicit.cconv1d(np.swapaxes(fT_o, -1, -2), np.swapaxes(gT_o, -1, -2))
        out = implicit.fftpad_forward(np.swapaxes(re, -1, -2), np.swapaxes(ro, -1, -2))
        return np.swapaxes(out, -1, -2)

    @staticmethod
    def cconv3d(f, g):
        """Function cconv3: fftpadBackward along x for every (j,k),
        cconv2 on every x-residue slab, fftpadForward along x."""
        f, g = _c(f), _c(g)
        fx = np.moveaxis(f, 0, -1)
        gx = np.moveaxis(g, 0, -1)
        fe, fo = implicit.fftpad_backward(fx)
        ge, go = implicit.fftpad_backward(gx)
        se = implicit.cconv2d(np.moveaxis(fe, -1, 0), np.moveaxis(ge, -1, 0))
        so = implicit.cconv2d(np.moveaxis(fo, -1, 0), np.moveaxis(go, -1, 0))
        out = implicit.fftpad_forward(np.moveaxis(se, 0, -1), np.moveaxis(so, 0, -1))
        return np.moveaxis(out, -1, 0)

    @staticmethod
    def hconv2d(f, g):
        """Function conv2: fft0padBackward on every column (centered
        x), Hermitian conv on every row of the three x-residue streams,
        fft0padForward on every column."""
        f, g = _c(f), _c(g)
        nx, my = f.shape
        mx = (nx + 1) // 2
        Sf = implicit.fft0pad_backward(f.T)   # r -> (my, mx): stream over l for each column ky
        Sg = implicit.fft0pad_backward(g.T)
        out_streams = {}
        for r in (-1, 0, 1):
            rows = implicit.hconv1d(Sf[r].T, Sg[r].T)   # (mx rows l, my)
            out_streams[r] = rows.T
        return implicit.fft0pad_forward(out_streams, mx).T

    @staticmethod
    def hconv3d(f, g):
        """Hermitian 3D "in an analogous manner", AMB-9: fft0pad
        along x, conv2 (hconv2d) on every x-residue slab, fft0pad forward."""
        f, g = _c(f), _c(g)
        nx, ny, mz = f.shape
        mx = (nx + 1) // 2
        Sf = implicit.fft0pad_backward(np.moveaxis(f, 0, -1))   # (ny, mz, mx)
        Sg = implicit.fft0pad_backward(np.moveaxis(g, 0, -1))
        out = {}
        for r in (-1, 0, 1):
            a = np.moveaxis(Sf[r], -1, 0)
            b = np.moveaxis(Sg[r], -1, 0)
            res = np.stack([implicit.hconv2d(a[l], b[l]) for l in range(mx)], axis=0)
            out[r] = np.moveaxis(res, 0, -1)
        return np.moveaxis(implicit.fft0pad_forward(out, mx), -1, 0)


# ================================================ O5 pseudospectral application ==

class application:
    """The 2D pseudospectral use case of P:859-876 written out as sums."""

    @staticmethod
    def hermitian_full2d(A):
        """(2mx-1, my) centered Hermitian storage -> (2mx-1, 2my-1) full array,
        ky = 0 line projected (AMB-7), U_{kx,-ky} = conj(U_{-kx,ky})."""
        A = _c(A).copy()
        nx, my = A.shape
        A[:, 0] = 0.5 * (A[:, 0] + np.conj(A[::-1, 0]))
        full = np.zeros((nx, 2 * my - 1), dtype=np.complex128)
        full[:, my - 1:] = A
        full[:, :my - 1] = np.conj(A[::-1, :0:-1])
        return full

    @staticmethod
    def euler_sum(w):
        """S_k = sum_p (p_x k_y - p_y k_x) / |k-p|^2 w_p w_{k-p}, p and
        k-p over the full centered range, 1/|q|^2 := 0 at q = 0 (no mean flow,
        S:398); output kx in [-mx+1, mx-1], ky in [0, my-1] (AMB-6).  Plain loops
        over k, numpy over p: small sizes only."""
        W = application.hermitian_full2d(w)
        nx, ny = W.shape
        mx, my = (nx + 1) // 2, (ny + 1) // 2
        px = np.arange(-(mx - 1), mx)[:, None]
        py = np.arange(-(my - 1), my)[None, :]
        out = np.zeros((nx, my), dtype=np.complex128)
        for kx in range(-(mx - 1), mx):
            for ky in range(0, my):
                qx, qy = kx - px, ky - py                       # k - p
                ok = (np.abs(qx) <= mx - 1) & (np.abs(qy) <= my - 1)
                q2 = (qx * qx + qy * qy).astype(np.float64)
                inv = np.where((q2 > 0) & ok, 1.0 / np.where(q2 > 0, q2, 1.0), 0.0)
                Wq = np.where(ok, W[np.clip(qx + mx - 1, 0, nx - 1), np.clip(qy + my - 1, 0, ny - 1)], 0.0)
                term = (px * ky - py * kx) * inv * W * Wq
                out[kx + mx - 1, ky] = term.sum()
        return out


    @staticmethod
    def euler_sum_at(w, idx):
        """S_k of euler_sum at the given linear output indices of
        the (2mx-1, my) storage, for large sizes: for each k the sum over p is
        taken over the rectangle where both p and k - p lie in the centered
        box (the same terms euler_sum masks), with numpy array slices."""
        W = application.hermitian_full2d(w)
        nx, ny = W.shape
        mx, my = (nx + 1) // 2, (ny + 1) // 2
        out = np.empty(len(idx), dtype=np.complex128)
        for o, lin in enumerate(np.asarray(idx, dtype=np.int64)):
            kx, ky = int(lin) // my - (mx - 1), int(lin) % my
            # p in [lo, hi] per axis with |p| <= m-1 and |k - p| <= m-1
            px0, px1 = max(-(mx - 1), kx - (mx - 1)), min(mx - 1, kx + (mx - 1))
            py0, py1 = max(-(my - 1), ky - (my - 1)), min(my - 1, ky + (my - 1))
            if px0 > px1 or py0 > py1:
                out[o] = 0.0
                continue
            px = np.arange(px0, px1 + 1)[:, None]
            py = np.arange(py0, py1 + 1)[None, :]
            Wp = W[px0 + mx - 1: px1 + mx, py0 + my - 1: py1 + my]
            # W_{k-p}: rows kx - px, columns ky - py, i.e. a reversed slice
            Wq = W[kx - px0 + mx - 1: kx - px1 + mx - 2 if kx - px1 + mx - 2 >= 0 else None: -1,
                   ky - py0 + my - 1: ky - py1 + my - 2 if ky - py1 + my - 2 >= 0 else None: -1]
            qx, qy = kx - px, ky - py
            q2 = (qx * qx + qy * qy).astype(np.float64)
            inv = np.where(q2 > 0, 1.0 / np.where(q2 > 0, q2, 1.0), 0.0)
            out[o] = ((px * ky - py * kx) * inv * Wp * Wq).sum()
        return out


# ===================================================== O1b 2D ternary (NEXT-2) ==

class ternary2d:
    """The 2D centered Hermitian ternary convolution of Function tconv2
    (P:962-964 in two dimensions), written as sums."""

    @staticmethod
    def full(A):
        """(2mx, my) paper layout (row 0 = kx -mx, ignored) -> full centered
        (2mx-1, 2my-1) array with U_{kx,-ky} = conj U_{-kx,ky} and the ky = 0
        line projected (AMB-7)."""
        return application.hermitian_full2d(_c(A)[1:])

    @staticmethod
    def direct(f, g, h):
        """t_k = sum_{p+q+r=k} f_p g_q h_r over the Hermitian-extended arrays
        (|px|,|qx|,|rx| <= mx-1, |py|,|qy|,|ry| <= my-1), two stages of direct 2D
        linear convolution (scipy.signal.convolve2d, method 'direct'); output in
        the paper layout (2mx, my): row i = kx i - mx, row 0 = 0, ky in [0, my)."""
        from scipy.signal import convolve2d
        F, G, H = ternary2d.full(f), ternary2d.full(g), ternary2d.full(h)
        nx, ny = F.shape
        mx, my = (nx + 1) // 2, (ny + 1) // 2
        e = convolve2d(F, G, mode="full")                 # indices p+q, origin (2mx-2, 2my-2)
        t = convolve2d(e, H, mode="full")                 # origin (3mx-3, 3my-3)
        ox, oy = 3 * (mx - 1), 3 * (my - 1)
        out = np.zeros((2 * mx, my), dtype=np.complex128)
        out[1:] = t[ox - (mx - 1):ox + mx, oy:oy + my]
        return out

    @staticmethod
    def brute(f, g, h):
        """Same sum by plain loops over all (p, q) with r = k - p - q (tiny sizes)."""
        F, G, H = ternary2d.full(f), ternary2d.full(g), ternary2d.full(h)
        nx, ny = F.shape
        mx, my = (nx + 1) // 2, (ny + 1) // 2
        out = np.zeros((2 * mx, my), dtype=np.complex128)
        for kx in range(-(mx - 1), mx):
            for ky in range(my):
                acc = 0j
                for px in range(-(mx - 1), mx):
                    for py in range(-(my - 1), my):
                        for qx in range(-(mx - 1), mx):
                            for qy in range(-(my - 1), my):
                                rx, ry = kx - px - qx, ky - py - qy
                                if abs(rx) <= mx - 1 and abs(ry) <= my - 1:
                                    acc += F[px + mx - 1, py + my - 1] * G[qx + mx - 1, qy + my - 1] * \
                                        H[rx + mx - 1, ry + my - 1]
                out[kx + mx, ky] = acc
        return out


# ======================================================== O4 closed forms ==

class closed:
    """O4: exact families.  The 1D ones are the paper's own test cases."""

    F_C = np.sqrt(3) + 1j * np.sqrt(7)
    G_C = np.sqrt(5) + 1j * np.sqrt(11)
    F_H = np.sqrt(3)
    G_H = np.sqrt(5)

    @staticmethod
    def cconv1d_inputs(m, F=None, G=None):
        F = closed.F_C if F is None else F
        G = closed.G_C if G is None else G
        k = np.arange(m)
        e = np.exp(1j * k)
        return F * e, G * e

    @staticmethod
    def cconv1d(m, F=None, G=None):
        """H_k = FG (k+1) e^{ik}."""
        F = closed.F_C if F is None else F
        G = closed.G_C if G is None else G
        k = np.arange(m)
        return F * G * (k + 1) * np.exp(1j * k)

    @staticmethod
    def hconv1d(m, F=None, G=None):
        """H_k = FG (2m-1-k) e^{ik}, F, G real."""
        F = closed.F_H if F is None else F
        G = closed.G_H if G is None else G
        k = np.arange(m)
        return F * G * (2 * m - 1 - k) * np.exp(1j * k)

    @staticmethod
    def ternary_count(m, k):
        """#{(p,q,r): p+q+r = k, |p|,|q|,|r| <= m-1} by inclusion-exclusion:
        sum_j (-1)^j C(3,j) C(n - j(2m-1) + 2, 2), n = k + 3(m-1), terms with
        n - j(2m-1) < 0 dropped (derived from P:963-964)."""
        from math import comb
        k = np.asarray(k)
        out = np.zeros(k.shape, dtype=np.float64)
        for idx, kk in np.ndenumerate(k):
            n = int(kk) + 3 * (m - 1)
            s = 0
            for j in range(4):
                t = n - j * (2 * m - 1)
                if t >= 0:
                    s += (-1) ** j * comb(3, j) * comb(t + 2, 2)
            out[idx] = s
        return out

    @staticmethod
    def tconv1d(m, F=1.0, G=1.0, H=1.0):
        """f_p = F e^{ip} etc. (F, G, H real) => t_k = FGH e^{ik} C(m,k)."""
        k = np.arange(m)
        return F * G * H * np.exp(1j * k) * closed.ternary_count(m, k)

    @staticmethod
    def cconv_nd(shape, F=None, G=None):
        """f = F e^{i sum k}, g = G e^{i sum k} => FG prod(k_a+1) e^{i sum k}."""
        F = closed.F_C if F is None else F
        G = closed.G_C if G is None else G
        grids = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
        ksum = sum(grids)
        f = F * np.exp(1j * ksum)
        g = G * np.exp(1j * ksum)
        cnt = np.ones(shape)
        for gr in grids:
            cnt = cnt * (gr + 1)
        return f, g, F * G * cnt * np.exp(1j * ksum)

    @staticmethod
    def hconv_nd(ms, F=None, G=None):
        """Centered axes ms[:-1] (storage 2m-1, k = i-(m-1)), Hermitian last axis
        (storage m, k = index); f = F e^{i sum k} with F real =>
        h = FG prod_centered(2m-1-|k|) * (2m_last-1-k_last) e^{i sum k}."""
        F = closed.F_H if F is None else F
        G = closed.G_H if G is None else G
        axes = [np.arange(-(m - 1), m) for m in ms[:-1]] + [np.arange(ms[-1])]
        grids = np.meshgrid(*axes, indexing="ij")
        ksum = sum(grids)
        f = F * np.exp(1j * ksum)
        g = G * np.exp(1j * ksum)
        cnt = np.ones(grids[0].shape)
        for m, gr in zip(ms, grids):
            cnt = cnt * (2 * m - 1 - np.abs(gr))
        return f.astype(np.complex128), g.astype(np.complex128), F * G * cnt * np.exp(1j * ksum)


def rel_l2(h, H) -> float:
    """Normalized L2 error sqrt(sum|h-H|^2)/sqrt(sum|H|^2)."""
    h = np.asarray(h)
    H = np.asarray(H)
    den = np.sqrt(np.sum(np.abs(H) ** 2))
    num = np.sqrt(np.sum(np.abs(h - H) ** 2))
    return float(num / den) if den > 0 else float(num)


# ======================================= workspace (memory) formulas ==

class memory:
    """Complex-word counts of the paper's implicit and explicit methods
    (P:766-769)."""

    @staticmethod
    def cconv2d_implicit(mx, my):
        return 4 * mx * my + 2 * my

    @staticmethod
    def cconv2d_explicit(mx, my):
        return 8 * mx * my

    @staticmethod
    def hconv2d_implicit(mx, my):
        return 2 * (2 * mx - 1) * my + 2 * (mx + 1) * my + 2 * (my // 2 + 1)

    @staticmethod
    def hconv2d_explicit(mx, my):
        return 2 * (3 * mx - 2) * (3 * my // 2)

    @staticmethod
    def cconv3d_implicit(mx, my, mz):
        return 4 * mx * my * mz + 2 * my * mz + 2 * mz

    @staticmethod
    def hconv3d_implicit(mx, my, mz):
        return 6 * mx * (2 * my - 1) * mz + 2 * (my + 1) * mz + 2 * (mz // 2 + 1)

    @staticmethod
    def tconv1d_implicit(m):
        return 6 * (m + 1)
