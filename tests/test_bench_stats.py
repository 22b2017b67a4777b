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


def test_gpus2_dry_run_spawns_two_ranks():
    """bench.py --gpus 2 launched directly re-launches itself under
    torch.distributed.run with two ranks (gloo rendezvous on 127.0.0.1)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=240, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["dry_run"] and d["world_size"] == 2 and len(set(d["rank_pids"])) == 2


def test_kernel_models_and_roofline_attribution():
    """Per-kernel algorithmic models and the attribution of
    overlapping kernel times to the step."""
    pk = bench.peaks()
    b, f = bench.kernel_model("K7", 512)
    assert b == 16 * (5 * 512 - 1) and math.isclose(f, 3 * 5 * 512 * 9)
    b, f = bench.kernel_model("K3", 512)
    assert b == 48 * 512 and math.isclose(f, 9 * 2.5 * 512 * 9)
    # two kernels of 30 ms each in a 40 ms step: overlap 1.5, each attributed 20 ms
    prof = [dict(tag="K3", n=512, launches=10, units=1000, ms=30.0),
            dict(tag="K7", n=512, launches=10, units=500, ms=30.0)]
    kt = bench.kernel_table(dict(bench.CONFIGS["c5b"], name="c5b"), prof, 1, pk, {}, 40.0)
    assert all(math.isclose(k["ms_attributed"], 20.0) for k in kt)
    assert math.isclose(kt[0]["overlap"], 1.5)
    r = bench.dominant_roofline(kt, pk)
    assert r["unit"] in ("GB/s", "TFLOP/s") and 0 < r["frac"]


def test_outputs_per_conv():
    assert bench.outputs_per_conv(bench.CONFIGS["c5b"]) == 1023 * 1023 * 512
    assert bench.outputs_per_conv(bench.CONFIGS["c1"]) == 1024
    assert bench.outputs_per_conv(bench.CONFIGS["c3b"]) == 256 * 256


def test_cpu_baseline_every_default_part():
    """Every config of the default run (except the two 3D ones, whose inputs
    are several GB) gets a CPU-oracle baseline: the sampler knows its kind."""
    names = [n for n in bench.DEFAULT_PARTS.split(",") if n not in ("c5a", "c5b")]
    assert "c4adv" in names and "c4t" in names
    for n in names:
        cb = bench.cpu_baseline(n, 0.01)
        assert cb["value"] > 0 and cb["unit"] == "conv/s" and cb["kind"] == "oracle", (n, cb)
        if n in ("c4adv", "c4t", "c3a", "c4"):
            assert "EXTRAPOLATED" in cb["sample"], (n, cb["sample"])
    for k in ("c5a", "c5b"):
        assert bench.CONFIGS[k]["kind"] in ("cconv3d", "hconv3d")
