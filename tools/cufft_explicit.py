"""Explicitly zero-padded convolutions on cuFFT (torch.fft) -- a COMPARISON
baseline only (BASELINE.json north_star: "an explicitly
padded cuFFT convolution may be timed only as a comparison baseline").  None
of this is on the product path.

The paper's explicit method: pad each input
with zeros to N = 2m (complex axes), N = 3m (centered / Hermitian axes, the
2/3 rule) or N = 4m (ternary), transform, multiply pointwise, transform back
and keep the dealiased range.  Hermitian axes use real (c2r / r2c)
transforms, which also project the input onto its Hermitian part (AMB-7),
exactly like the implicit method.

    python tools/cufft_explicit.py            # time every config, compare with idconv
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

F = torch.fft


def cconv1d(f, g):
    m = f.shape[-1]
    return F.ifft(F.fft(f, n=2 * m) * F.fft(g, n=2 * m))[..., :m]


def _half_pad(U, N):
    """Half spectrum k = 0..m-1 of a Hermitian axis, zero-padded to N//2 + 1."""
    m = U.shape[-1]
    P = torch.zeros(U.shape[:-1] + (N // 2 + 1,), dtype=U.dtype, device=U.device)
    P[..., :m] = U
    return P


def hconv1d(f, g):
    m = f.shape[-1]
    N = 3 * m
    u = F.irfft(_half_pad(f, N), n=N) * N
    v = F.irfft(_half_pad(g, N), n=N) * N
    return F.rfft(u * v)[..., :m] / N


def tconv1d(f, g, h):
    m = f.shape[-1]
    N = 4 * m
    u = F.irfft(_half_pad(f, N), n=N) * N
    u *= F.irfft(_half_pad(g, N), n=N) * N
    u *= F.irfft(_half_pad(h, N), n=N) * N
    return F.rfft(u)[..., :m] / N


def cconv2d(f, g):
    mx, my = f.shape[-2:]
    s = (2 * mx, 2 * my)
    return F.ifft2(F.fft2(f, s=s) * F.fft2(g, s=s))[..., :mx, :my]


def _centered_pad(A, axes_m, N_axes, herm_N):
    """Place centered axes (index i <-> k = i - (m-1)) at k mod N; the last axis
    is a Hermitian half axis padded to herm_N // 2 + 1."""
    shape = tuple(N_axes) + (herm_N // 2 + 1,)
    P = torch.zeros(A.shape[:-len(shape)] + shape, dtype=A.dtype, device=A.device)
    idx = []
    for m, N in zip(axes_m, N_axes):
        k = torch.arange(-(m - 1), m, device=A.device)
        idx.append(k % N)
    mz = A.shape[-1]
    if len(axes_m) == 1:
        P[..., idx[0], :mz] = A
    else:
        P[..., idx[0][:, None], idx[1][None, :], :mz] = A
    return P, idx


def hconv2d(f, g):
    nx, my = f.shape
    mx = (nx + 1) // 2
    Nx, Ny = 3 * mx, 3 * my
    Pf, idx = _centered_pad(f, (mx,), (Nx,), Ny)
    u = F.irfft2(Pf, s=(Nx, Ny)) * (Nx * Ny)
    del Pf
    Pg, _ = _centered_pad(g, (mx,), (Nx,), Ny)
    u *= F.irfft2(Pg, s=(Nx, Ny)) * (Nx * Ny)
    del Pg
    H = F.rfft2(u) / (Nx * Ny)
    return H[idx[0], :my]


def tconv2d(f, g, h):
    """2D centered Hermitian ternary (Function tconv2's problem): paper layout
    (2mx, my), row 0 = kx -mx ignored; pad x to 4mx (centered), y to 4my
    (Hermitian half), three c2r, product, r2c."""
    nx, my = f.shape
    mx = nx // 2
    Nx, Ny = 4 * mx, 4 * my
    u = None
    for a in (f, g, h):
        P, idx = _centered_pad(a[1:], (mx,), (Nx,), Ny)
        x = F.irfft2(P, s=(Nx, Ny)) * (Nx * Ny)
        del P
        u = x if u is None else u * x
    H = F.rfft2(u) / (Nx * Ny)
    out = torch.zeros_like(f)
    out[1:] = H[idx[0], :my]
    return out


# ---- pruned explicit versions ----------
# Johnson's pruning: transform first along the axes whose padded
# half is zero, so that the later (outer) transforms skip the all-zero lines;
# the inverse transforms run in the opposite order and drop the unneeded half
# before the next axis.  Same padded sizes, same results, fewer transforms.

def cconv2d_pruned(f, g):
    """y-pruned explicit 2D complex: x transforms only on the my
    unpadded columns, both ways."""
    mx, my = f.shape[-2:]

    def fwd(a):
        return F.fft(F.fft(a, n=2 * mx, dim=-2), n=2 * my, dim=-1)
    X = fwd(f)
    X *= fwd(g)
    return F.ifft(F.ifft(X, dim=-1)[..., :my], dim=-2)[..., :mx, :]


def _centered_rows(A, m, N):
    """Centered axis -2 (index i <-> k = i - (m-1)) placed at k mod N."""
    k = torch.arange(-(m - 1), m, device=A.device) % N
    P = torch.zeros(A.shape[:-2] + (N, A.shape[-1]), dtype=A.dtype, device=A.device)
    P[..., k, :] = A
    return P, k


def hconv2d_pruned(f, g):
    """y-pruned explicit 2D centered Hermitian: complex x transforms (3mx) on
    the my stored half-spectrum columns only, then c2r along y (3my)."""
    nx, my = f.shape
    mx = (nx + 1) // 2
    Nx, Ny = 3 * mx, 3 * my

    def bwd(a):
        P, k = _centered_rows(a, mx, Nx)
        return F.irfft(F.ifft(P, dim=0) * Nx, n=Ny, dim=1) * Ny, k
    u, k = bwd(f)
    w, _ = bwd(g)
    u *= w
    del w
    return F.fft(F.rfft(u, dim=1)[:, :my], dim=0)[k] / (Nx * Ny)


def tconv2d_pruned(f, g, h):
    """y-pruned explicit 2D centered Hermitian ternary: 4mx x
    4my padding, x transforms on the my stored columns only."""
    nx, my = f.shape
    mx = nx // 2
    Nx, Ny = 4 * mx, 4 * my
    u = None
    for a in (f, g, h):
        P, k = _centered_rows(a[1:], mx, Nx)
        x = F.irfft(F.ifft(P, dim=0) * Nx, n=Ny, dim=1) * Ny
        del P
        u = x if u is None else u * x
    H = F.fft(F.rfft(u, dim=1)[:, :my], dim=0)[k] / (Nx * Ny)
    out = torch.zeros_like(f)
    out[1:] = H
    return out


def cconv3d_pruned(f, g):
    """Pruned explicit 3D complex (the paper's xz-pruned comparison,
    P:884-886, pruned on every axis it can be): z transforms on the mx*my
    stored lines, y on mx*2mz, x on 2my*2mz; inverses in reverse order."""
    mx, my, mz = f.shape

    def fwd(a):
        return F.fft(F.fft(F.fft(a, n=2 * mz, dim=2), n=2 * my, dim=1), n=2 * mx, dim=0)
    X = fwd(f)
    X *= fwd(g)
    X = F.ifft(X, dim=0)[:mx]
    X = F.ifft(X, dim=1)[:, :my]
    return F.ifft(X, dim=2)[..., :mz]


def cconv3d(f, g):
    mx, my, mz = f.shape
    s = (2 * mx, 2 * my, 2 * mz)
    X = F.fftn(f, s=s)
    X *= F.fftn(g, s=s)
    return F.ifftn(X)[:mx, :my, :mz]


def hconv3d(f, g):
    nx, ny, mz = f.shape
    mx, my = (nx + 1) // 2, (ny + 1) // 2
    Nx, Ny, Nz = 3 * mx, 3 * my, 3 * mz
    Pf, idx = _centered_pad(f, (mx, my), (Nx, Ny), Nz)
    u = F.irfftn(Pf, s=(Nx, Ny, Nz)) * (Nx * Ny * Nz)
    del Pf
    Pg, _ = _centered_pad(g, (mx, my), (Nx, Ny), Nz)
    u *= F.irfftn(Pg, s=(Nx, Ny, Nz)) * (Nx * Ny * Nz)
    del Pg
    H = F.rfftn(u) / (Nx * Ny * Nz)
    del u
    return H[idx[0][:, None], idx[1][None, :], :mz]


CONFIGS = [  # (name, kind, shape, arrays) -- BASELINE.json configs
    ("c1", "cconv1d", (32768, 1024), 2),
    ("c2a", "hconv1d", (4096, 4096), 2),
    ("c2b", "tconv1d", (4096, 4096), 3),
    ("c3a", "cconv2d", (1024, 1024), 2),
    ("c3b", "cconv2d", (64, 256, 256), 2),
    ("c4", "hconv2d", (4095, 2048), 2),
    ("c4t", "tconv2d", (4096, 2048), 3),
    ("c5a", "cconv3d", (512, 512, 512), 2),
    ("c5b", "hconv3d", (1023, 1023, 512), 2),
]


PRUNED = {"cconv2d": cconv2d_pruned, "hconv2d": hconv2d_pruned, "tconv2d": tconv2d_pruned,
          "cconv3d": cconv3d_pruned}


def _time(fn, reps=3):
    """Best of `reps` timed calls (after one warm-up) and the peak device
    memory the call allocates beyond what is live before it (bytes)."""
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    out = fn()
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    for a, b in ev:
        a.record()
        out = fn()
        b.record()
    torch.cuda.synchronize()
    return min(a.elapsed_time(b) for a, b in ev), out, peak


def _run(fn):
    try:
        t, out, peak = _time(fn)
        return t, out.clone(), peak, None
    except torch.OutOfMemoryError as e:
        return None, None, None, "out of memory: " + str(e).splitlines()[0]
    finally:
        torch.cuda.empty_cache()


def main():
    from paper_1008_1366_b200 import idconv
    import synthgen
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for name, kind, shape, narr in CONFIGS:
        if a.only and name not in a.only.split(","):
            continue
        arrs = [torch.empty(shape, dtype=torch.complex128, device="cuda") for _ in range(narr)]
        for i, x in enumerate(arrs):
            idconv.fill_uniform(x, synthgen.array_id(i), synthgen.SEED)
            if kind == "tconv2d":
                x[0] = 0                                   # kx = -mx row
        batched = kind == "cconv2d" and len(shape) == 3

        def call(fn):   # the 2D complex functions are batched over leading axes
            return lambda: fn(*arrs)
        explicit = {"cconv1d": cconv1d, "hconv1d": hconv1d, "tconv1d": tconv1d, "cconv2d": cconv2d,
                    "hconv2d": hconv2d, "tconv2d": tconv2d, "cconv3d": cconv3d, "hconv3d": hconv3d}[kind]
        t_ex, ref, mem_ex, ex_err = _run(call(explicit))
        t_pr = mem_pr = pr_err = None
        diff_pr = None
        if kind in PRUNED:
            t_pr, out_pr, mem_pr, pr_err = _run(call(PRUNED[kind]))
            if out_pr is not None and ref is not None:
                diff_pr = float(torch.linalg.vector_norm(out_pr - ref) / torch.linalg.vector_norm(ref))
            del out_pr
        pristine = [x.clone() for x in arrs]
        ws = idconv.workspace_bytes(getattr(idconv, kind.upper()), *_sizes(kind, shape),
                                    batch=shape[0] if batched else 1)
        # implicit timed without the restore copies
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = None
        for _ in range(4):
            for x, p in zip(arrs, pristine):
                x.copy_(p)
            torch.cuda.synchronize()
            ev0.record()
            getattr(idconv, kind)(*arrs)
            ev1.record()
            torch.cuda.synchronize()
            t = ev0.elapsed_time(ev1)
            best = t if best is None else min(best, t)
        diff = None
        if ref is not None:
            diff = float(torch.linalg.vector_norm(arrs[0] - ref) / torch.linalg.vector_norm(ref))
        in_bytes = sum(x.numel() * 16 for x in arrs)
        row = dict(config=name, kind=kind, shape=list(shape), explicit_cufft_ms=t_ex, implicit_ms=best,
                   speedup=(t_ex / best) if t_ex else None, rel_l2_implicit_vs_explicit=diff, error=ex_err,
                   pruned_cufft_ms=t_pr, speedup_vs_pruned=(t_pr / best) if t_pr else None,
                   rel_l2_pruned_vs_explicit=diff_pr, pruned_error=pr_err,
                   input_bytes=in_bytes, implicit_workspace_bytes=ws,
                   explicit_extra_bytes=mem_ex, pruned_extra_bytes=mem_pr)
        print(json.dumps(row), flush=True)
        rows.append(row)
        del arrs, pristine, ref
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(rows, fh, indent=1)


def _sizes(kind, shape):
    if kind in ("cconv1d", "hconv1d", "tconv1d"):
        return (shape[-1],)
    if kind == "cconv2d":
        return tuple(shape[-2:])
    if kind in ("hconv2d", "tconv2d"):
        return ((shape[0] + 1) // 2, shape[1])
    if kind == "cconv3d":
        return tuple(shape)
    return ((shape[0] + 1) // 2, (shape[1] + 1) // 2, shape[2])


if __name__ == "__main__":
    main()
