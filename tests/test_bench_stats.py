"""bench.py's timing statistics: the paper's one-sided standard deviations
(P:258-262 with the AMB-5 reading of the garbled root)."""
import math

import bench


def test_one_sided_sigmas():
    t = [1.0, 2.0, 3.0, 10.0]                 # mean 4
    s = bench.timing_stats(t)
    d = len(t) / 2 - 1                          # n/2 - 1 = 1
    assert s["mean_ms"] == 4.0 and s["median_ms"] == 2.5
    assert math.isclose(s["sigma_L_ms"], math.sqrt((9 + 4 + 1) / d))
    assert math.isclose(s["sigma_H_ms"], math.sqrt(36 / d))


def test_constant_samples_have_zero_spread():
    s = bench.timing_stats([2.0] * 6)
    assert s["sigma_L_ms"] == 0.0 and s["sigma_H_ms"] == 0.0
