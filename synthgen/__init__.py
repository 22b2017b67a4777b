"""Seeded, index-addressable synthetic inputs for the implicit-dealiasing hot path.

This module is the ONLY code shared between the oracle side (``oracle/``, the
tests) and the product side (``bench.py``).  It holds none of the method's
arithmetic: it draws numbers and applies the input recipe of the workloads
(SURVEY.md §8(c) c.2 / §8(d) d.1).

Generator ("Input generator"):

* ``sm(x)``  = splitmix64 finalizer (all arithmetic mod 2**64)::

      z = x + 0x9E3779B97F4A7C15
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
      z = (z ^ (z >> 27)) * 0x94D049BB133111EB
      return z ^ (z >> 31)

* stream key ``s = sm(seed ^ sm(array_id))``, ``array_id = role + 4*item``
  (role f=0, g=1, h=2);
* value ``x = sm(s + 2*linear_index + part)`` (part 0 = Re, 1 = Im), mapped to
  ``((x >> 11) * 2**-53) * 2 - 1`` in [-1, 1).

The CUDA library carries an independent implementation of the same counter
generator (``idc_fill_uniform``); tests check the two bitwise.

Recipes (BASELINE.json configs; SURVEY AMB-17):

* complex kinds: Re, Im iid U[-1, 1);
* Hermitian kinds: Im U_0 := 0 (1D);
  2D: scaled by 1/(1 + kx^2 + ky^2), kx = i - (mx-1) (centered), ky = j;
  the ky = 0 line is made conjugate-symmetric by overwriting kx < 0 with
  conj(U[-kx, 0]); U_00 real.
  3D: scaled by 1/(1+kx^2+ky^2+kz^2) (kx, ky centered, kz = index);
  kz = 0 plane symmetrised by overwriting (kx<0) u (kx=0, ky<0) with the
  conjugate of the mirror (-kx, -ky); U_000 real.
* complex 3D: scaled by 1/(1 + kx^2 + ky^2 + kz^2) with k = index.
"""
from __future__ import annotations

import numpy as np

SEED = 10081366
ROLE_F, ROLE_G, ROLE_H = 0, 1, 2

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_C0 = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def sm_scalar(x: int) -> int:
    """splitmix64 finalizer on a Python int (reference scalar form)."""
    m = (1 << 64) - 1
    z = (int(x) + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def sm(x: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer, vectorised over uint64 (wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64, copy=False) + _C0
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        return z ^ (z >> np.uint64(31))


def stream_key(seed: int, array_id: int) -> int:
    return sm_scalar(int(seed) ^ sm_scalar(int(array_id)))


def uniform_complex(n: int, array_id: int, seed: int = SEED, start: int = 0) -> np.ndarray:
    """n complex128 values, Re/Im iid U[-1,1), for linear indices start..start+n-1."""
    s = np.uint64(stream_key(seed, array_id))
    idx = np.arange(start, start + n, dtype=np.uint64)
    out = np.empty(n, dtype=np.complex128)
    with np.errstate(over="ignore"):
        base = s + np.uint64(2) * idx
        for part in (0, 1):
            x = sm(base + np.uint64(part))
            v = (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0
            if part == 0:
                out.real = v
            else:
                out.imag = v
    return out


def uniform_at(array_id: int, linear_index: int, seed: int = SEED) -> complex:
    """Single value (scalar path), for index-addressable sampling and golden checks."""
    s = stream_key(seed, array_id)
    vals = []
    for part in (0, 1):
        x = sm_scalar((s + 2 * int(linear_index) + part) & ((1 << 64) - 1))
        vals.append((x >> 11) * (2.0 ** -53) * 2.0 - 1.0)
    return complex(vals[0], vals[1])


def array_id(role: int, item: int = 0) -> int:
    return role + 4 * item


# ---------------------------------------------------------------- recipes ---

def cconv1d_inputs(m: int, batch: int = 1, roles=(ROLE_F, ROLE_G), seed: int = SEED):
    """Config 1 shape: (batch, m) complex128 per role, iid U[-1,1) parts."""
    outs = []
    for role in roles:
        a = np.empty((batch, m), dtype=np.complex128)
        for b in range(batch):
            a[b] = uniform_complex(m, array_id(role, b), seed)
        outs.append(a)
    return outs


def hconv1d_inputs(m: int, batch: int = 1, roles=(ROLE_F, ROLE_G), seed: int = SEED):
    """Config 2 shape: (batch, m) complex128, k = 0..m-1, Im f_0 := 0."""
    outs = cconv1d_inputs(m, batch, roles, seed)
    for a in outs:
        a[:, 0] = a[:, 0].real
    return outs


def cconv2d_inputs(mx: int, my: int, batch: int = 1, roles=(ROLE_F, ROLE_G), seed: int = SEED):
    """Config 3 shape: (batch, mx, my) complex128, iid U[-1,1) parts."""
    outs = []
    for role in roles:
        a = np.empty((batch, mx, my), dtype=np.complex128)
        for b in range(batch):
            a[b] = uniform_complex(mx * my, array_id(role, b), seed).reshape(mx, my)
        outs.append(a)
    return outs


def hermitian2d_symmetrize(a: np.ndarray) -> np.ndarray:
    """Make the ky=0 line of a (2mx-1, my) centered array conjugate-symmetric
    by overwriting kx<0 with conj(U[-kx,0]); U_00 := Re U_00 (AMB-17)."""
    nx = a.shape[0]
    mx = (nx + 1) // 2
    c = mx - 1
    for kx in range(1, mx):
        a[c - kx, 0] = np.conj(a[c + kx, 0])
    a[c, 0] = a[c, 0].real
    return a


def hconv2d_inputs(mx: int, my: int, roles=(ROLE_F, ROLE_G), seed: int = SEED, scaled: bool = True):
    """Config 4 shape: (2mx-1, my), scaled by 1/(1+kx^2+ky^2), ky=0 line symmetric."""
    nx = 2 * mx - 1
    kx = (np.arange(nx) - (mx - 1)).astype(np.float64)
    ky = np.arange(my).astype(np.float64)
    k2 = kx[:, None] ** 2 + ky[None, :] ** 2
    outs = []
    for role in roles:
        a = uniform_complex(nx * my, array_id(role, 0), seed).reshape(nx, my)
        if scaled:
            a = a / (1.0 + k2)
        outs.append(hermitian2d_symmetrize(a))
    return outs


def cconv3d_inputs(mx: int, my: int, mz: int, roles=(ROLE_F, ROLE_G), seed: int = SEED, scaled: bool = True):
    """Config 5a shape: (mx, my, mz), scaled by 1/(1+kx^2+ky^2+kz^2), k = index."""
    kx = np.arange(mx, dtype=np.float64)
    ky = np.arange(my, dtype=np.float64)
    kz = np.arange(mz, dtype=np.float64)
    k2 = kx[:, None, None] ** 2 + ky[None, :, None] ** 2 + kz[None, None, :] ** 2
    outs = []
    for role in roles:
        a = uniform_complex(mx * my * mz, array_id(role, 0), seed).reshape(mx, my, mz)
        if scaled:
            a = a / (1.0 + k2)
        outs.append(a)
    return outs


def hermitian3d_symmetrize(a: np.ndarray) -> np.ndarray:
    """kz=0 plane of a (2mx-1, 2my-1, mz) centered array made conjugate-symmetric:
    overwrite (kx<0) u (kx=0, ky<0) with conj(U[-kx,-ky,0]); U_000 real."""
    nx, ny = a.shape[0], a.shape[1]
    cx, cy = (nx - 1) // 2, (ny - 1) // 2
    p = a[:, :, 0]
    # kx < 0 half-plane: rows 0..cx-1 mirror rows nx-1..cx+1, columns reversed
    p[:cx, :] = np.conj(p[nx - 1:cx:-1, ::-1])
    # kx = 0, ky < 0
    p[cx, :cy] = np.conj(p[cx, ny - 1:cy:-1])
    p[cx, cy] = p[cx, cy].real
    a[:, :, 0] = p
    return a


def hconv3d_inputs(mx: int, my: int, mz: int, roles=(ROLE_F, ROLE_G), seed: int = SEED, scaled: bool = True):
    """Config 5b shape: (2mx-1, 2my-1, mz), scaled by 1/(1+|k|^2), kz=0 plane symmetric."""
    nx, ny = 2 * mx - 1, 2 * my - 1
    kx = (np.arange(nx) - (mx - 1)).astype(np.float64)
    ky = (np.arange(ny) - (my - 1)).astype(np.float64)
    kz = np.arange(mz, dtype=np.float64)
    k2 = kx[:, None, None] ** 2 + ky[None, :, None] ** 2 + kz[None, None, :] ** 2
    outs = []
    for role in roles:
        a = uniform_complex(nx * ny * mz, array_id(role, 0), seed).reshape(nx, ny, mz)
        if scaled:
            a = a / (1.0 + k2)
        outs.append(hermitian3d_symmetrize(a))
    return outs
