"""GPU parity of the 1D kinds against the oracle.

Element-by-element relative L2 error against the oracle's direct
sums on the same seeded inputs, gate 1e-12 (BASELINE.json north_star); every
power-of-two m from 1 to 8192 with ragged batches (not a multiple of the
rows-per-CTA), the paper's exact families, and the full-size configs sampled
row by row.  Calls go through the C ABI (paper_1008_1366_b200.idconv)."""
import numpy as np
import pytest
import torch

import oracle
import synthgen
from oracle import closed, direct, rel_l2

pytestmark = pytest.mark.gpu
GATE = 1e-12
MS = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192]


@pytest.fixture(scope="module")
def idc():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1008_1366_b200 import idconv
    return idconv


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def batch_for(m):
    # ragged: 3 rows for big m, more for small m, never a multiple of the rows per CTA
    return 3 if m >= 2048 else (7 if m >= 256 else 37)


@pytest.mark.parametrize("m", MS)
def test_cconv1d_random(idc, m):
    B = batch_for(m)
    f, g = synthgen.cconv1d_inputs(m, B)
    ref = direct.cconv1d(f, g)
    F, G = dev(f), dev(g)
    idc.cconv1d(F, G)
    err = rel_l2(F.cpu().numpy(), ref)
    assert err < GATE, err
    assert err < 1e-14, err   # expected rounding floor ~1e-15 (SURVEY c.5)


@pytest.mark.parametrize("m", MS)
def test_hconv1d_random(idc, m):
    B = batch_for(m)
    f, g = synthgen.hconv1d_inputs(m, B)
    ref = direct.hconv1d(f, g)
    F, G = dev(f), dev(g)
    idc.hconv1d(F, G)
    err = rel_l2(F.cpu().numpy(), ref)
    assert err < 1e-14, err


@pytest.mark.parametrize("m", MS)
def test_tconv1d_random(idc, m):
    B = 2 if m >= 2048 else batch_for(m)
    f, g, h = synthgen.hconv1d_inputs(m, B, roles=(0, 1, 2))
    ref = direct.tconv1d(f, g, h)
    F, G, H = dev(f), dev(g), dev(h)
    idc.tconv1d(F, G, H)
    err = rel_l2(F.cpu().numpy(), ref)
    assert err < 1e-14, err


def test_hermitian_projection_imag_dc_ignored(idc):
    """AMB-7: Im f_0 is discarded; the GPU must not depend on it."""
    m = 64
    f, g = synthgen.cconv1d_inputs(m, 5)       # Im f_0 != 0 on purpose
    ref = direct.hconv1d(f, g)                  # oracle projects f_0 := Re f_0
    F, G = dev(f), dev(g)
    idc.hconv1d(F, G)
    assert rel_l2(F.cpu().numpy(), ref) < 1e-14


@pytest.mark.parametrize("m", [8, 1024, 4096])
def test_paper_families(idc, m):
    f, g = closed.cconv1d_inputs(m)
    F, G = dev(f[None]), dev(g[None])
    idc.cconv1d(F, G)
    assert rel_l2(F.cpu().numpy()[0], closed.cconv1d(m)) < 1e-14
    k = np.arange(m)
    F, G = dev((np.sqrt(3) * np.exp(1j * k))[None]), dev((np.sqrt(5) * np.exp(1j * k))[None])
    idc.hconv1d(F, G)
    assert rel_l2(F.cpu().numpy()[0], closed.hconv1d(m)) < 1e-14
    e = np.exp(1j * k)[None]
    F, G, H = dev(np.sqrt(3) * e), dev(np.sqrt(5) * e), dev(np.sqrt(2) * e)
    idc.tconv1d(F, G, H)
    assert rel_l2(F.cpu().numpy()[0], closed.tconv1d(m, np.sqrt(3), np.sqrt(5), np.sqrt(2))) < 1e-14


def test_special_cases(idc):
    m = 16
    top = np.zeros((1, m), complex)
    top[0, m - 1] = 1
    F, G = dev(top), dev(top)
    idc.cconv1d(F, G)
    assert np.max(np.abs(F.cpu().numpy())) < 1e-15        # top mode does not alias (D1)
    F, G = dev(top), dev(top)
    idc.hconv1d(F, G)
    out = F.cpu().numpy()[0]
    assert abs(out[0] - 2) < 1e-14 and np.max(np.abs(out[1:])) < 1e-14
    F, G, H = dev(top), dev(top), dev(top)
    idc.tconv1d(F, G, H)
    out = F.cpu().numpy()[0]
    assert abs(out[m - 1] - 3) < 1e-14 and np.max(np.abs(out[:m - 1])) < 1e-14


def test_device_generator_bitwise(idc):
    for aid, start, n in [(0, 0, 1000), (5, 4095, 17), (4 * 300 + 1, 12345, 4096)]:
        out = torch.empty(n, dtype=torch.complex128, device="cuda")
        idc.fill_uniform(out, aid, synthgen.SEED, start)
        ref = synthgen.uniform_complex(n, aid, start=start)
        assert np.array_equal(out.cpu().numpy(), ref)


def test_host_tensors_end_to_end(idc):
    m, B = 256, 5
    f, g = synthgen.cconv1d_inputs(m, B)
    F = torch.from_numpy(f.copy()).pin_memory()
    G = torch.from_numpy(g.copy()).pin_memory()
    idc.cconv1d(F, G)
    torch.cuda.synchronize()
    assert rel_l2(F.numpy(), direct.cconv1d(f, g)) < 1e-14


def test_repeated_calls_and_workspace_reuse(idc):
    m, B = 8192, 2
    f, g = synthgen.cconv1d_inputs(m, B)
    ref = direct.cconv1d(f, g)
    for _ in range(2):
        F, G = dev(f), dev(g)
        idc.cconv1d(F, G)
        assert rel_l2(F.cpu().numpy(), ref) < 1e-14


# ----------------------------------------------------- full-size configs --

def device_inputs(m, B, roles, hermitian):
    arrs = []
    for role in roles:
        a = torch.empty((B, m), dtype=torch.complex128, device="cuda")
        for b in range(B):  # one stream per batch item (array_id = role + 4*item)
            pass
        arrs.append(a)
    from paper_1008_1366_b200 import idconv
    for role, a in zip(roles, arrs):
        for b in range(B):
            idconv.fill_uniform(a[b], synthgen.array_id(role, b), synthgen.SEED)
        if hermitian:
            a[:, 0] = a[:, 0].real.to(torch.complex128)
    return arrs


def sampled_rows(B, n, seed=7):
    rs = np.random.default_rng(seed)
    return np.unique(np.concatenate([[0, B - 1], rs.choice(B, n, replace=False)]))


def test_config1_cconv1d_full(idc):
    """C1: m = 1024, B = 32768 at full size; 34 sampled rows vs direct sums."""
    m, B = 1024, 32768
    F, G = device_inputs(m, B, (0, 1), False)
    rows = sampled_rows(B, 32)
    idc.cconv1d(F, G)
    out = F[torch.from_numpy(rows).cuda()].cpu().numpy()
    f, g = (np.stack([synthgen.uniform_complex(m, synthgen.array_id(r, b)) for b in rows]) for r in (0, 1))
    assert rel_l2(out, direct.cconv1d(f, g)) < 1e-14


def test_config2_hconv_tconv_full(idc):
    """C2: hconv1d and tconv1d at m = 4096, B = 4096 (the bench launch); sampled rows."""
    m, B = 4096, 4096
    rows = sampled_rows(B, 14)
    F, G = device_inputs(m, B, (0, 1), True)
    idc.hconv1d(F, G)
    out = F[torch.from_numpy(rows).cuda()].cpu().numpy()
    f, g = (np.stack([synthgen.uniform_complex(m, synthgen.array_id(r, b)) for b in rows]) for r in (0, 1))
    f[:, 0] = f[:, 0].real
    g[:, 0] = g[:, 0].real
    assert rel_l2(out, direct.hconv1d(f, g)) < 1e-14
    del F, G
    rows = sampled_rows(B, 4)
    F, G, H = device_inputs(m, B, (0, 1, 2), True)
    idc.tconv1d(F, G, H)
    out = F[torch.from_numpy(rows).cuda()].cpu().numpy()
    f, g, h = (np.stack([synthgen.uniform_complex(m, synthgen.array_id(r, b)) for b in rows]) for r in (0, 1, 2))
    for a in (f, g, h):
        a[:, 0] = a[:, 0].real
    assert rel_l2(out, direct.tconv1d(f, g, h)) < 1e-14
