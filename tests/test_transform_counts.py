"""Transform-count invariant (tests/golden/paper_examples.json
"transform_counts"): the number of size-m transforms each convolution runs,
counted on the device by the debug build libidconv_count.so (the product
kernels compiled with -DIDC_COUNT_FFT=1: every executed FFT adds 1 to
counter[log2 N]).

Paper counts per 1D convolution: Function
cconv 6 complex transforms of size m; the centered Hermitian conv 9 real
transforms of size m; Function tconv 8 real transforms of size 2m.  This
implementation: cconv 6 complex FFT(m) -- the paper's count; hconv 5 complex
FFT(m) -- the 9 real transforms packed two per complex FFT (f + i g, p_0 +
i p_1) and the tenth half carrying p_{-1} alone; tconv
8 complex FFT(m) -- the 4-residue split of DESIGN.md section 6, the same
8 m log m work as the paper's 8 real FFT(2m).  2D: Function cconv2 / conv2
 -- 6 my FFT(mx) along x and 6 FFT(my) on each of the 2mx
residue rows (cconv2); 9 my FFT(mx) and 5 FFT(my) on each of the 3mx
residue rows (conv2)."""
import ctypes
import json
import os

import numpy as np
import pytest
import torch

import synthgen
from oracle import direct, rel_l2

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def clib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1008_1366_b200 import idconv
    path = os.path.join(ROOT, "paper_1008_1366_b200", "libidconv_count.so")
    if not os.path.exists(path):
        pytest.fail("libidconv_count.so missing: __graft_entry__.build() builds it")
    L = ctypes.CDLL(path)
    for name, (args, res) in idconv.SIGNATURES.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


def counts(L, fn):
    assert L.idc_fft_count_begin() == 0
    assert fn() == 0
    out = (ctypes.c_ulonglong * 16)()
    assert L.idc_fft_count_end(out) == 0
    return {1 << i: int(out[i]) for i in range(16) if out[i]}


def P(t):
    return ctypes.c_void_p(t.data_ptr())


def work(kind, m0, m1=1, m2=1, batch=1):
    """(pointer, bytes) of a workspace for the call (the m = 8192 rows need one)."""
    from paper_1008_1366_b200 import idconv
    nb = idconv.workspace_bytes(kind, m0, m1, m2, batch)
    w = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")
    work.keep = w
    return P(w), nb


GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_examples.json")))["transform_counts"]


def real_equivalents(complex_ffts_of_m, m_paper_size_ratio=1):
    """Complex FFT(m) counted on the device -> the paper's real transforms
    (one complex transform = two real ones of the same size, or one real
    transform of twice the size for tconv)."""
    return 2 * complex_ffts_of_m if m_paper_size_ratio == 1 else complex_ffts_of_m


# batches are whole row groups of the kernels (rows per CTA: 256 at m = 4, 32
# at m = 64, 4 at m = 512 and 1024, 1 from 4096): the counter counts every
# executed transform, including those of padding groups of a partial CTA
@pytest.mark.parametrize("m,B", [(4, 256), (64, 32), (512, 8), (1024, 4), (4096, 2), (8192, 2)])
def test_cconv1d_six_transforms(clib, m, B):
    f, g = synthgen.cconv1d_inputs(m, B)
    F, G = torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()
    from paper_1008_1366_b200 import idconv
    wp, nb = work(idconv.CCONV1D, m, batch=B)
    c = counts(clib, lambda: clib.idc_cconv1d(P(F), P(G), m, B, wp, nb, None))
    assert c == {m: 6 * B}, c
    assert c[m] // B == GOLDEN["cconv"]                          # six complex transforms of size m
    assert rel_l2(F.cpu().numpy(), direct.cconv1d(f, g)) < 1e-14   # the debug build computes the same result


@pytest.mark.parametrize("m,B", [(4, 256), (64, 32), (512, 8), (1024, 4), (4096, 2)])
def test_hconv1d_nine_real_transforms(clib, m, B):
    f, g = synthgen.hconv1d_inputs(m, B)
    F, G = torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()
    from paper_1008_1366_b200 import idconv
    wp, nb = work(idconv.HCONV1D, m, batch=B)
    c = counts(clib, lambda: clib.idc_hconv1d(P(F), P(G), m, B, wp, nb, None))
    # 9 real transforms = 4.5 complex; packed: 5 complex FFT(m) per row,
    # i.e. one real transform more than the paper (p_{-1} alone in a complex FFT)
    assert c == {m: 5 * B}, c
    assert real_equivalents(c[m] // B) == GOLDEN["hconv"] + 1
    assert rel_l2(F.cpu().numpy(), direct.hconv1d(f, g)) < 1e-14


@pytest.mark.parametrize("m,B", [(4, 256), (64, 32), (512, 4), (4096, 2)])
def test_tconv1d_eight_transforms(clib, m, B):
    f, g, h = synthgen.hconv1d_inputs(m, B, roles=(0, 1, 2))
    F, G, H = (torch.from_numpy(a).cuda() for a in (f, g, h))
    from paper_1008_1366_b200 import idconv
    wp, nb = work(idconv.TCONV1D, m, batch=B)
    c = counts(clib, lambda: clib.idc_tconv1d(P(F), P(G), P(H), m, B, wp, nb, None))
    # 8 real FFT(2m) == 8 complex FFT(m) of the 4-residue split
    assert c == {m: 8 * B}, c
    assert real_equivalents(c[m] // B, 2) == GOLDEN["tconv"]
    assert rel_l2(F.cpu().numpy(), direct.tconv1d(f, g, h)) < 1e-14


@pytest.mark.parametrize("mx,my", [(64, 32), (512, 16), (256, 256)])
def test_cconv2d_counts(clib, mx, my):
    from paper_1008_1366_b200 import idconv
    f, g = synthgen.cconv2d_inputs(mx, my, 1)
    F, G = torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()
    nb = idconv.workspace_bytes(idconv.CCONV2D, mx, my, 1, 1)
    Wk = torch.empty(nb, dtype=torch.uint8, device="cuda")
    c = counts(clib, lambda: clib.idc_cconv2d(P(F), P(G), mx, my, 1, P(Wk), nb, None))
    want = {}
    want[mx] = want.get(mx, 0) + 6 * my                          # x: 2 inputs x 2 streams + 2 forward
    want[my] = want.get(my, 0) + 2 * mx * 6                      # rows of both x-streams
    assert c == want, c


@pytest.mark.parametrize("mx,my", [(64, 512), (16, 1024), (32, 512)])
def test_hconv2d_counts(clib, mx, my):
    from paper_1008_1366_b200 import idconv
    f, g = synthgen.hconv2d_inputs(mx, my)
    F, G = torch.from_numpy(f).cuda(), torch.from_numpy(g).cuda()
    nb = idconv.workspace_bytes(idconv.HCONV2D, mx, my, 1, 1)
    Wk = torch.empty(nb, dtype=torch.uint8, device="cuda")
    c = counts(clib, lambda: clib.idc_hconv2d(P(F), P(G), mx, my, P(Wk), nb, None))
    want = {}
    want[mx] = want.get(mx, 0) + 9 * my                          # x: 2 inputs x 3 streams + 3 forward
    want[my] = want.get(my, 0) + 3 * mx * 5                      # 3mx residue rows, 5 complex FFT(my)
    assert c == want, c


def test_product_library_has_no_counter():
    from paper_1008_1366_b200 import idconv
    assert idconv.lib().idc_fft_count_begin() == idconv.ERR_UNSUPPORTED
