"""Memory accounting (tools/memory_report.py): the
paper's word counts as transcribed, and this implementation's inputs +
workspace (idc_workspace_bytes, a host-side query of the C ABI) against them."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import memory_report as mr  # noqa: E402


@pytest.mark.parametrize("mx,my,mz", [(2, 2, 2), (4, 8, 16), (512, 512, 512), (2048, 1024, 4)])
def test_paper_formulas_match_their_stated_closed_forms(mx, my, mz):
    # each left side is the paper's itemised count, the right side the
    # simplified form the paper prints next to it
    imp, exp = mr.paper_words("hconv2d", mx, my)
    assert imp == 6 * mx * my + my + 2
    assert exp == 2 * (3 * mx - 2) * (3 * my // 2)             # P:783 "2(3mx-2)(3my/2) = 9mxmy-6my"
    imp, exp = mr.paper_words("tconv2d", mx, my)
    assert imp == 12 * mx * my + 12 * mx + 3 * my + 3
    assert exp == 24 * mx * my + 12 * mx
    imp, _ = mr.paper_words("hconv3d", mx, my, mz)
    # P:894's printed right side is 2mz short of its itemised left side
    # (AMB-21); the report uses the itemised count
    assert imp == 12 * mx * my * mz - 6 * mx * mz + 2 * my * mz + mz + 2 + 2 * mz
    imp, exp = mr.paper_words("tconv1d", mx)
    assert (imp, exp) == (6 * mx + 6, 6 * mx + 3)


def test_asymptotic_ratios():
    # implicit/explicit -> 1/2 (2D complex), 1/4 (3D complex),
    # 2/3 (2D Hermitian), 4/9 (3D Hermitian) as m -> infinity
    m = 1 << 20
    r = lambda k, *s: (lambda p: p[0] / p[1])(mr.paper_words(k, *s))
    assert abs(r("cconv2d", m, m) - 1 / 2) < 1e-5
    assert abs(r("hconv2d", m, m) - 2 / 3) < 1e-5
    m = 1 << 12
    assert abs(r("cconv3d", m, m, m) - 1 / 4) < 1e-3
    assert abs(r("hconv3d", m, m, m) - 4 / 9) < 1e-3


def test_implementation_memory_against_the_paper():
    rows = {r["config"]: r for r in mr.report(None)}
    for name, r in rows.items():
        if r["kind"].endswith("1d"):
            # rows are fused in registers: no work arrays beyond the inputs
            assert r["ours_total_words"] <= r["paper_implicit_words"]
        else:
            # 2D/3D: never above explicit padding; 2D within 0.5% of the
            # paper's implicit count (3D slab groups trade some memory for
            # launch granularity)
            assert r["ours_total_words"] < r["paper_explicit_words"]
            if r["kind"].endswith("2d"):
                assert r["ours_total_words"] <= 1.005 * r["paper_implicit_words"]
            else:
                assert r["ours_total_words"] <= 1.25 * r["paper_implicit_words"]
