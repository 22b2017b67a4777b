"""The explicitly padded comparison baseline (tools/cufft_explicit.py, SURVEY
8(f) NEXT-4) computes the same dealiased convolutions: checked against the
oracle's direct sums on small inputs (torch.fft on the CPU here; the same
functions run on cuFFT in the comparison run)."""
import os
import sys

import numpy as np
import pytest
import torch

import synthgen
from oracle import direct, rel_l2

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import cufft_explicit as ex  # noqa: E402


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a))


def test_explicit_1d():
    f, g, h = synthgen.hconv1d_inputs(32, 3, roles=(0, 1, 2))
    assert rel_l2(ex.cconv1d(T(f), T(g)).numpy(), direct.cconv1d(f, g)) < 1e-14
    assert rel_l2(ex.hconv1d(T(f), T(g)).numpy(), direct.hconv1d(f, g)) < 1e-14
    assert rel_l2(ex.tconv1d(T(f), T(g), T(h)).numpy(), direct.tconv1d(f, g, h)) < 1e-14


@pytest.mark.parametrize("shape", [(8, 16), (16, 4)])
def test_explicit_2d(shape):
    f, g = synthgen.cconv2d_inputs(*shape, 2)
    ref = np.stack([direct.cconv2d(f[b], g[b]) for b in range(2)])
    assert rel_l2(ex.cconv2d(T(f), T(g)).numpy(), ref) < 1e-14
    f, g = synthgen.hconv2d_inputs(*shape)
    assert rel_l2(ex.hconv2d(T(f), T(g)).numpy(), direct.hconv2d(f, g)) < 1e-14


def test_explicit_3d():
    f, g = synthgen.cconv3d_inputs(4, 8, 4)
    assert rel_l2(ex.cconv3d(T(f), T(g)).numpy(), direct.cconv3d(f, g)) < 1e-14
    f, g = synthgen.hconv3d_inputs(4, 4, 4)
    assert rel_l2(ex.hconv3d(T(f), T(g)).numpy(), direct.hconv3d(f, g)) < 1e-14


def test_explicit_tconv2d():
    from oracle import ternary2d
    mx, my = 4, 8
    arrs = []
    for r in range(3):
        a = synthgen.hconv2d_inputs(mx, my, roles=(r,))[0]
        arrs.append(np.concatenate([np.zeros((1, my), dtype=np.complex128), a], axis=0))
    assert rel_l2(ex.tconv2d(*(T(a) for a in arrs)).numpy(), ternary2d.direct(*arrs)) < 1e-14


@pytest.mark.parametrize("shape", [(8, 16), (16, 4)])
def test_pruned_2d(shape):
    """Pruned explicit versions: same padded sizes, the
    zero lines skipped -- must equal the oracle's direct sums."""
    f, g = synthgen.cconv2d_inputs(*shape, 2)
    ref = np.stack([direct.cconv2d(f[b], g[b]) for b in range(2)])
    assert rel_l2(ex.cconv2d_pruned(T(f), T(g)).numpy(), ref) < 1e-14
    f, g = synthgen.hconv2d_inputs(*shape)
    assert rel_l2(ex.hconv2d_pruned(T(f), T(g)).numpy(), direct.hconv2d(f, g)) < 1e-14


def test_pruned_3d_and_ternary():
    from oracle import ternary2d
    f, g = synthgen.cconv3d_inputs(4, 8, 4)
    assert rel_l2(ex.cconv3d_pruned(T(f), T(g)).numpy(), direct.cconv3d(f, g)) < 1e-14
    mx, my = 4, 8
    arrs = []
    for r in range(3):
        a = synthgen.hconv2d_inputs(mx, my, roles=(r,))[0]
        arrs.append(np.concatenate([np.zeros((1, my), dtype=np.complex128), a], axis=0))
    assert rel_l2(ex.tconv2d_pruned(*(T(a) for a in arrs)).numpy(), ternary2d.direct(*arrs)) < 1e-14
