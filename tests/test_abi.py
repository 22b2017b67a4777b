"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/idconv.h declares, and rejects bad arguments synchronously
before touching the device (include/idconv.h "Errors")."""
import ctypes
import os
import re

import pytest

from paper_1008_1366_b200 import idconv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "idconv.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"IDC_API\s+[\w\s\*]+?\b(idc_\w+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ["idc_cconv1d", "idc_hconv1d", "idc_tconv1d", "idc_cconv2d", "idc_hconv2d", "idc_cconv3d",
                 "idc_hconv3d", "idc_workspace_bytes", "idc_status_string"]:
        assert name in syms


def test_library_exports_every_declared_symbol():
    L = idconv.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
        assert name in idconv.SIGNATURES, name


def test_exports_match_nm():
    out = os.popen(f"nm -D --defined-only {idconv.LIB_PATH}").read()
    exported = set(re.findall(r"\bT (idc_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_version_and_status_strings():
    assert "sm_100a" in idconv.version()
    for code in range(6):
        assert idconv.status_string(code).startswith("IDC_")


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {idconv.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_sass_no_tensor_core_ops_and_tma_present():
    """the path is not a dense contraction, so no
    tensor-core instruction (HMMA / DMMA / IMMA / UTC*MMA) may appear in the
    library; the pencil and row kernels move tiles with TMA (UTMALDG /
    UTMASTG tensor copies, UBLKCP bulk copies)."""
    import collections
    import re
    sass = os.popen(f"/usr/local/cuda/bin/cuobjdump -sass {idconv.LIB_PATH} 2>&1").read()
    ops = collections.Counter(re.findall(r"\b(HMMA|DMMA|IMMA|UTCHMMA|UTCQMMA|UTCIMMA|UTCMMA|UTMALDG|UTMASTG|UBLKCP)\b", sass))
    assert sum(ops[k] for k in ("HMMA", "DMMA", "IMMA", "UTCHMMA", "UTCQMMA", "UTCIMMA", "UTCMMA")) == 0, ops
    assert ops["UTMALDG"] > 0 and ops["UTMASTG"] > 0 and ops["UBLKCP"] > 0, ops
    assert len(re.findall(r"\bDFMA\b", sass)) > 1000


def _fake(addr):
    return ctypes.c_void_p(addr)


@pytest.mark.parametrize("m", [0, 3, 12, 16384])
def test_bad_sizes_rejected(m):
    L = idconv.lib()
    code = L.idc_cconv1d(_fake(0x1000), _fake(0x100000), m, 1, None, 0, None)
    assert code == (idconv.ERR_INVALID if m == 0 else idconv.ERR_UNSUPPORTED)
    code = L.idc_hconv1d(_fake(0x1000), _fake(0x100000), m, 1, None, 0, None)
    assert code == (idconv.ERR_INVALID if m == 0 else idconv.ERR_UNSUPPORTED)


def test_null_misaligned_aliasing_batch0():
    L = idconv.lib()
    assert L.idc_cconv1d(None, _fake(0x100000), 16, 1, None, 0, None) == idconv.ERR_INVALID
    assert L.idc_cconv1d(_fake(0x1008), _fake(0x100000), 16, 1, None, 0, None) == idconv.ERR_INVALID
    # f and g overlap: 16 complex = 256 bytes each
    assert L.idc_cconv1d(_fake(0x1000), _fake(0x1080), 16, 1, None, 0, None) == idconv.ERR_INVALID
    assert L.idc_cconv1d(_fake(0x1000), _fake(0x100000), 16, 0, None, 0, None) == idconv.ERR_INVALID
    assert L.idc_tconv1d(_fake(0x1000), _fake(0x2000), _fake(0x1000), 16, 1, None, 0, None) == idconv.ERR_INVALID


def test_workspace_queries():
    # 1D rows keep their work vectors on chip up to m = 4096 (P:374-377 u, v live in smem/registers)
    for m in [1, 2, 64, 1024, 4096]:
        assert idconv.workspace_bytes(idconv.CCONV1D, m) == 0
        assert idconv.workspace_bytes(idconv.HCONV1D, m) == 0
        assert idconv.workspace_bytes(idconv.TCONV1D, m) == 0
    assert idconv.workspace_bytes(idconv.CCONV1D, 8192) > 0
    assert idconv.workspace_bytes(idconv.CCONV1D, 3) == 0


def test_workspace_too_small_is_reported():
    L = idconv.lib()
    need = idconv.workspace_bytes(idconv.CCONV1D, 8192)
    assert L.idc_cconv1d(_fake(0x1000), _fake(0x10000000), 8192, 1, _fake(0x40000000), need - 16, None) \
        == idconv.ERR_WORKSPACE
    # workspace aliasing f
    assert L.idc_cconv1d(_fake(0x1000), _fake(0x10000000), 8192, 1, _fake(0x1000), need, None) \
        == idconv.ERR_INVALID


def test_no_cpu_fallback():
    """The product path refuses CPU execution when no GPU exists (no fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    f = torch.zeros(4, dtype=torch.complex128)
    with pytest.raises(Exception):
        idconv.cconv1d(f, f.clone())


def test_launch_count_is_monotonic_without_gpu():
    n0 = idconv.launch_count()
    assert n0 >= 0 and idconv.launch_count() == n0          # no launches without calls


@pytest.mark.gpu
def test_launch_count_counts_hot_path_kernels():
    import torch
    f = torch.zeros((3, 64), dtype=torch.complex128, device="cuda")
    g = torch.zeros_like(f)
    n0 = idconv.launch_count()
    idconv.cconv1d(f, g)                                     # one fused row kernel
    assert idconv.launch_count() - n0 == 1
    a = torch.zeros((16, 16), dtype=torch.complex128, device="cuda")
    b = torch.zeros_like(a)
    n1 = idconv.launch_count()
    idconv.cconv2d(a, b)                                     # K5, K2 (both x-streams), K6
    assert idconv.launch_count() - n1 == 3


@pytest.mark.gpu
def test_profiler_reports_kernel_classes_and_units():
    """idc_profile_begin/end: one record per kernel class with launches, units
    (rows / pencil columns) and a positive device time."""
    import torch
    a = torch.zeros((2, 64, 32), dtype=torch.complex128, device="cuda")
    b = torch.zeros_like(a)
    idconv.profile_begin()
    idconv.cconv2d(a, b)                                     # K5 (64 cols x 2 items x 2 inputs), K2, K6
    recs = {r["tag"]: r for r in idconv.profile_end()}
    assert set(recs) == {"K5", "K2", "K6"} or set(recs) == {"K5s", "K2", "K6s"}, recs
    k5 = recs.get("K5") or recs["K5s"]
    assert k5["n"] == 64 and k5["units"] == 32 * 2 * 2 and k5["launches"] == 1
    assert recs["K2"]["n"] == 32 and recs["K2"]["units"] == 2 * 2 * 64
    assert all(r["ms"] > 0 for r in recs.values())
    again = {r["tag"]: r for r in idconv.profile_end()}              # a second end returns the same window
    assert again == recs
