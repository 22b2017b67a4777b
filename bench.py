#!/usr/bin/env python
"""Benchmark of the implicitly dealiased convolution hot path on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` prints ONE
JSON line on rank 0.

Headline (``value``): config 5b -- the 3D centered Hermitian convolution
hconv3d of 512^3 modes, (2*512-1)^2 x 512 complex128 arrays, the largest
single-GPU configuration of BASELINE.json.  One step = one idc_hconv3d call
(every row of SURVEY 8(a): the x-pencil fft0pad backward, the per-x-residue
slab 2D convolutions -- y pencils, z rows -- and the forward passes), inputs
resident in HBM.  Every other config (C1 cconv1d, C2a hconv1d, C2b tconv1d,
C3a / C3b cconv2d, C4 hconv2d, C5a cconv3d) and the two §8(f) NEXT calls at
the C4 size (c4adv: the 2D Euler advective term, c4t: the 2D ternary
tconv2d) are measured the same way and reported in ``parts``, each with its
own roofline, kernel table, host-buffer e2e and CPU-oracle baseline.

Timing: W warm-up calls, then K timed calls, each bracketed by CUDA events on
the launch stream; before every call (outside the events) the inputs are
restored from pristine device copies (the call is in place) and a 256 MB
buffer is written (L2 flush).  The library's per-kernel-class event profiler
(idc_profile_begin/end) runs over a second pass of the same K calls right
after the timed loop (its per-launch events serialise the launches and would
add ~15% to a 0.1 ms call if they ran inside it) and gives each kernel's
device time, from which the dominant kernel's achieved algorithmic bytes or
flops per launch are computed (``roofline``).

Multi-GPU (``--gpus N``; under torchrun, or self-spawned through
torch.distributed.run when launched directly): the headline becomes ONE
config-5b convolution slab-sharded over the N ranks (idc_hconv3d_dist: y
pencils, ncclAlltoAll, per-residue (x, z) convolutions, ncclAlltoAll back;
"scaling": "strong"); C5a likewise through idc_cconv3d_dist; the 1D/2D
configs are independent problems -> replicas on every rank ("weak").
Times are device times, max over ranks.

``--impl reference`` times the CPU oracle (oracle/: direct sums, the
reference arm of this tier) on the host cores on a bounded sample of the
headline workload per step, extrapolated to whole convolutions.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synthgen  # noqa: E402  (seeded inputs; no method arithmetic)

METRIC = "dealiased convolutions/sec (fp64) and achieved HBM GB/s vs B200 peak"
W = 16  # bytes per complex128 word
HEADLINE = "c5b"
DEFAULT_PARTS = "c1,c2a,c2b,c3a,c3b,c4,c5a,c4adv,c4t"


def peaks():
    """Roofline denominators: HBM from MEASURED_PEAKS.json (driver-written),
    fp64 from the unit count x max clock."""
    src = "MEASURED_PEAKS.json"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            hbm = float(json.load(fh)["hbm_gbs"])
    except Exception:
        src = "fallback 6650 (B200_PROFILING.md)"
        hbm = 6650.0
    # 148 SMs x 64 fp64 FMA lanes x 2 flop x 1.965 GHz (measured DFMA loop: 34.2 TF/s, profiles/r01_peaks.txt)
    fp64 = 148 * 64 * 2 * 1.965e9 / 1e12
    return {"hbm_gbs": hbm, "hbm_src": src, "fp64_tflops": fp64,
            "fp64_src": "148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz (DESIGN.md); measured DFMA loop 34.2"}


# ------------------------------------------------------------------ configs --

def flops_rfft(n):      # 2.5 n log2 n per real transform
    return 2.5 * n * np.log2(n) if n > 1 else 0.0


def flops_cfft(n):      # 5 n log2 n per complex transform
    return 5.0 * n * np.log2(n) if n > 1 else 0.0


CONFIGS = {
    "c1": dict(kind="cconv1d", m=1024, batch=32768, narr=2, desc="configs[0] C1: cconv1d m=1024, B=32768 rows"),
    "c2a": dict(kind="hconv1d", m=4096, batch=4096, narr=2, desc="configs[1] C2a: hconv1d m=4096, B=4096 rows"),
    "c2b": dict(kind="tconv1d", m=4096, batch=4096, narr=3, desc="configs[1] C2b: tconv1d m=4096, B=4096 rows"),
    "c3a": dict(kind="cconv2d", m=(1024, 1024), batch=1, narr=2, desc="configs[2] C3a: cconv2d 1024x1024"),
    "c3b": dict(kind="cconv2d", m=(256, 256), batch=64, narr=2, desc="configs[2] C3b: cconv2d 64 x 256x256"),
    "c4": dict(kind="hconv2d", m=(2048, 2048), batch=1, narr=2,
               desc="configs[3] C4: hconv2d mx=my=2048, (2mx-1) x my"),
    "c5a": dict(kind="cconv3d", m=(512, 512, 512), batch=1, narr=2, desc="configs[4] C5a: cconv3d 512^3"),
    "c5b": dict(kind="hconv3d", m=(512, 512, 512), batch=1, narr=2,
                desc="configs[4] C5b: hconv3d 512^3 modes, (2m-1)^2 x m"),
    # SURVEY 8(f) NEXT rows (not part of the default run)
    "c4adv": dict(kind="advection2d", m=(2048, 2048), batch=1, narr=2,
                  desc="NEXT-1: 2D Euler advective term (M=2 dot-product conv2, P:867-876), mx=my=2048"),
    "c4t": dict(kind="tconv2d", m=(2048, 2048), batch=1, narr=3,
                desc="NEXT-2: 2D centered Hermitian ternary (Function tconv2, P:1087-1109), mx=my=2048"),
}


def shape_of(p):
    m, k = p["m"], p["kind"]
    if k.endswith("1d"):
        return (p["batch"], m)
    if k == "cconv2d":
        return (p["batch"],) + tuple(m)
    if k in ("hconv2d", "advection2d"):
        return (2 * m[0] - 1, m[1])
    if k == "tconv2d":
        return (2 * m[0], m[1])
    if k == "cconv3d":
        return tuple(m)
    if k == "hconv3d":
        return (2 * m[0] - 1, 2 * m[1] - 1, m[2])
    raise ValueError(k)


def outputs_per_conv(p):
    """Output values of one convolution (for extrapolating sampled oracle sums)."""
    shp = shape_of(p)
    n = int(np.prod(shp))
    return n // p["batch"] if p["kind"] in ("cconv1d", "hconv1d", "tconv1d", "cconv2d") else n


def part_model(p):
    """Algorithmic HBM bytes and convention flops per convolution:
    bytes = the method's minimum traffic with one HBM round trip per dependent
    phase and per-row work on chip; flops = 5 n log2 n per complex FFT(n),
    2.5 n log2 n per real FFT(n), counted with the paper's transform counts."""
    m, kind = p["m"], p["kind"]
    if kind == "cconv1d":
        return 3 * W * m, 6 * flops_cfft(m)                 # 6 complex FFTs of size m
    if kind == "hconv1d":
        return 3 * W * m, 9 * flops_rfft(m)                 # 9 real FFTs of size m
    if kind == "tconv1d":
        return 4 * W * m, 8 * flops_rfft(2 * m)             # 8 real FFTs of size 2m
    if kind == "cconv2d":
        mx, my = m
        fl = 6 * my * flops_cfft(mx) + 2 * mx * 6 * flops_cfft(my)
        return 15 * W * mx * my, fl
    if kind == "hconv2d":
        mx, my = m
        fl = 9 * my * flops_cfft(mx) + 3 * mx * 9 * flops_rfft(my)
        return W * (3 * (2 * mx - 1) * my + 18 * mx * my), fl
    if kind == "advection2d":
        mx, my = m
        fl = 15 * my * flops_cfft(mx) + 3 * mx * 15 * flops_rfft(my)
        return W * (12 * (2 * mx - 1) * my + 30 * mx * my), fl
    if kind == "tconv2d":
        mx, my = m
        fl = 8 * my * flops_cfft(2 * mx) + 4 * mx * 8 * flops_rfft(2 * my)
        return 20 * W * 2 * mx * my, fl
    if kind == "cconv3d":
        mx, my, mz = m
        fl = 6 * my * mz * flops_cfft(mx) + 2 * mx * (6 * mz * flops_cfft(my) + 2 * my * 6 * flops_cfft(mz))
        return 15 * W * mx * my * mz, fl
    if kind == "hconv3d":
        mx, my, mz = m
        ny = 2 * my - 1
        fl = 9 * ny * mz * flops_cfft(mx) + 3 * mx * (9 * mz * flops_cfft(my) + 3 * my * 9 * flops_rfft(mz))
        return W * (3 * (2 * mx - 1) * ny * mz + 18 * mx * ny * mz), fl
    raise ValueError(kind)


# Per-kernel algorithmic model: bytes and convention
# flops per UNIT of a launch (a row for the row kernels, a column for the
# pencils), n = the kernel's transform size.
def kernel_model(tag, n):
    lg = np.log2(n) if n > 1 else 0.0
    base = tag.rstrip("s").replace("v1", "")
    if base == "K2":        # Function cconv per row: read f, g, write f; 6 FFT(m)
        return 3 * W * n, 6 * 5 * n * lg
    if base == "K3":        # centered Hermitian conv per row: 9 real FFT(m)
        return 3 * W * n, 9 * 2.5 * n * lg
    if base == "K4":        # ternary per row: read f, g, h, write f; 8 real FFT(2m)
        return 4 * W * n, 8 * 2.5 * 2 * n * np.log2(2 * n)
    if base == "K5":        # fftpadBackward per column: read m, write 2 streams of m; 2 FFT(m)
        return 3 * W * n, 2 * 5 * n * lg
    if base == "K6":        # fftpadForward per column: read 2m, write m
        return 3 * W * n, 2 * 5 * n * lg
    if base in ("K7", "K8"):  # fft0pad per column: 2m-1 <-> 3 streams of m; 3 FFT(m)
        return W * (5 * n - 1), 3 * 5 * n * lg
    return None, None


# ------------------------------------------------------------ GPU clocks --

class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 3 + i and r[3 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- helpers --

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def timing_stats(t):
    """Median and the paper's one-sided standard deviations of per-call times
    (AMB-5): sigma_L/H = sqrt(sum_{t_i < T / t_i > T} (t_i - T)^2 / (n/2 - 1)),
    T the mean of the n samples."""
    n = len(t)
    T = sum(t) / n
    d = max(n / 2 - 1, 1)
    lo = sum((x - T) ** 2 for x in t if x < T)
    hi = sum((x - T) ** 2 for x in t if x > T)
    return {"n": n, "mean_ms": T, "median_ms": statistics.median(t), "sigma_L_ms": (lo / d) ** 0.5,
            "sigma_H_ms": (hi / d) ** 0.5}


def load_traffic():
    """ncu DRAM bytes per unit of each kernel class (profiles/traffic.json,
    written by tools/collect_traffic.py from one `ncu --set full` capture)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def make_inputs(idc, torch, p, rank, dev):
    """Seeded device inputs for one config; batch
    item ids offset by rank (replicas at N > 1)."""
    kind, B, narr = p["kind"], p["batch"], p["narr"]
    if kind == "tconv2d":       # paper layout: a zero kx = -mx row, then the hconv2d recipe
        q = dict(p, kind="hconv2d")
        return [torch.cat([torch.zeros((1, a.shape[1]), dtype=a.dtype, device=dev), a], dim=0).contiguous()
                for a in make_inputs(idc, torch, q, rank, dev)]
    shp = shape_of(p)
    arrs = []
    for role in range(narr):
        a = torch.empty(shp, dtype=torch.complex128, device=dev)
        if kind.endswith("1d") or kind == "cconv2d":
            for b in range(B):              # one seeded stream per batch item (array_id = role + 4 item)
                idc.fill_uniform(a[b], synthgen.array_id(role, rank * B + b), synthgen.SEED)
        else:
            idc.fill_uniform(a, synthgen.array_id(role, rank), synthgen.SEED)
        if kind in ("hconv1d", "tconv1d"):
            a[:, 0] = a[:, 0].real.to(torch.complex128)   # Im U_0 := 0 (config 2)
        elif kind in ("hconv2d", "advection2d", "cconv3d", "hconv3d"):
            axes = []
            for d, n in enumerate(shp):
                k = torch.arange(n, device=dev, dtype=torch.float64)
                centered = (kind in ("hconv2d", "advection2d") and d == 0) or (kind == "hconv3d" and d < 2)
                if centered:
                    k = k - (n - 1) // 2
                axes.append(k)
            k2 = sum((ax ** 2).reshape([-1 if i == j else 1 for i in range(len(shp))]) for j, ax in enumerate(axes))
            a /= (1.0 + k2)
            del k2
            if kind in ("hconv2d", "advection2d"):     # ky = 0 line conjugate-symmetric, U_00 real
                c = (shp[0] - 1) // 2
                a[:c, 0] = torch.conj(torch.flip(a[c + 1:, 0], dims=(0,)))
                a[c, 0] = a[c, 0].real.to(torch.complex128)
            elif kind == "hconv3d":                    # kz = 0 plane conjugate-symmetric
                cx, cy = (shp[0] - 1) // 2, (shp[1] - 1) // 2
                pl = a[:, :, 0]
                pl[:cx, :] = torch.conj(torch.flip(pl[cx + 1:, :], dims=(0, 1)))
                pl[cx, :cy] = torch.conj(torch.flip(pl[cx, cy + 1:], dims=(0,)))
                pl[cx, cy] = pl[cx, cy].real.to(torch.complex128)
        arrs.append(a)
    return arrs


def make_dist_inputs(idc, torch, p, rank, ws, dev):
    """This rank's x-slab of the config-5 arrays (hconv3d: the 2mx-1 planes
    padded to 2mx with a zero plane), generated index-addressably with the
    config's 1/(1+|k|^2) scaling.  Timing input: the kz = 0 plane is not
    re-symmetrised across ranks (the call convolves its Hermitian projection,
    AMB-7; the arithmetic is the same)."""
    mx, my, mz = p["m"]
    herm = p["kind"] == "hconv3d"
    planes = 2 * mx if herm else mx
    nx = planes // ws
    x0 = rank * nx
    ny = 2 * my - 1 if herm else my
    plane = ny * mz
    out = []
    for role in range(2):
        a = torch.empty((nx, ny, mz), dtype=torch.complex128, device=dev)
        idc.fill_uniform(a, synthgen.array_id(role, 0), synthgen.SEED, start=x0 * plane)
        kx = torch.arange(x0, x0 + nx, device=dev, dtype=torch.float64) - ((mx - 1) if herm else 0)
        kyv = torch.arange(ny, device=dev, dtype=torch.float64) - ((my - 1) if herm else 0)
        kz = torch.arange(mz, device=dev, dtype=torch.float64)
        a /= 1.0 + kx[:, None, None] ** 2 + kyv[None, :, None] ** 2 + kz[None, None, :] ** 2
        if herm and x0 + nx == planes:
            a[-1].zero_()                                  # padding plane
        out.append(a)
    return out


def call(idc, p, arrs):
    if p["kind"] == "advection2d":                      # (w, out); device-only call
        if arrs[0].is_cuda:
            return idc.advection2d(arrs[0], out=arrs[1])
        out = idc.advection2d(arrs[0].to("cuda", non_blocking=True))
        arrs[0].copy_(out, non_blocking=True)
        return arrs[0]
    return getattr(idc, p["kind"])(*arrs)


def kernel_table(p, prof, steps, pk, traffic, step_ms):
    """Per-kernel-class device time of one call and its achieved algorithmic
    bytes / flops (DESIGN.md section 6 models).  The 3D calls run slab groups
    on concurrent streams, so their kernels' event times overlap and sum to
    more than the step; each kernel is then attributed its share of the step
    (ms_attributed = step x share), and achieved = its algorithmic bytes or
    flops / ms_attributed."""
    tot = sum(r["ms"] for r in prof) or 1.0
    overlap = max(1.0, tot / steps / step_ms)
    rows = []
    for r in prof:
        b_u, f_u = kernel_model(r["tag"], r["n"])
        d = dict(kernel=f"{r['tag']}<{r['n']}>", launches_per_call=r["launches"] / steps,
                 ms_per_call=r["ms"] / steps, share=r["ms"] / tot, units_per_launch=r["units"] / r["launches"],
                 ms_attributed=r["ms"] / steps / overlap, overlap=overlap)
        if b_u is not None:
            sec = r["ms"] / overlap / 1e3
            d["hbm_gbs_alg"] = b_u * r["units"] / sec / 1e9
            d["fp64_tflops_alg"] = f_u * r["units"] / sec / 1e12
            d["hbm_frac"] = d["hbm_gbs_alg"] / pk["hbm_gbs"]
            d["fp64_frac"] = d["fp64_tflops_alg"] / pk["fp64_tflops"]
            t_b = b_u / (pk["hbm_gbs"] * 1e9)
            t_f = f_u / (pk["fp64_tflops"] * 1e12)
            d["bound"] = "hbm" if t_b >= t_f else "alu"
            tpu = traffic.get(f"{p.get('name', '')}:{r['tag']}:{r['n']}") or traffic.get(f"{r['tag']}:{r['n']}")
            d["traffic_per_launch"] = tpu * d["units_per_launch"] if tpu else None
        rows.append(d)
    rows.sort(key=lambda d: -d["ms_per_call"])
    return rows


def dominant_roofline(kt, pk):
    """roofline object of the contract for the dominant kernel of a call."""
    for d in kt:
        if "bound" not in d:
            continue
        if d["bound"] == "hbm":
            r = {"bound": "hbm", "achieved": d["hbm_gbs_alg"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                 "peak_src": pk["hbm_src"]}
        else:
            r = {"bound": "alu", "achieved": d["fp64_tflops_alg"], "peak": pk["fp64_tflops"], "unit": "TFLOP/s",
                 "peak_src": pk["fp64_src"]}
        r["frac"] = r["achieved"] / r["peak"]
        r["traffic"] = d.get("traffic_per_launch")
        r["kernel"] = d["kernel"]
        r["share_of_step"] = d["share"]
        r["units_per_launch"] = d["units_per_launch"]
        r["hbm_frac"] = d["hbm_frac"]
        r["fp64_frac"] = d["fp64_frac"]
        return r
    return None


# -------------------------------------------------------------- our arm ----

def measure(idc, torch, tdist, name, args, rank, ws, dev, comm=None, want_e2e=False):
    """Time one config: W warm-up calls, K timed calls (restore + L2 flush
    before each, outside the events), kernel profile over a second pass of K calls."""
    p = dict(CONFIGS[name], name=name)
    dist3d = comm is not None and p["kind"] in ("cconv3d", "hconv3d")
    if dist3d:
        pristine = make_dist_inputs(idc, torch, p, rank, ws, dev)
        mx, my, mz = p["m"]
        fn = idc.hconv3d_dist if p["kind"] == "hconv3d" else idc.cconv3d_dist

        def run(arrs):
            fn(comm, arrs[0], arrs[1], mx, my, mz)
    else:
        pristine = make_inputs(idc, torch, p, rank, dev)

        def run(arrs):
            call(idc, p, arrs)
    work = [torch.empty_like(a) for a in pristine]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # 2x L2
    stream = torch.cuda.current_stream(dev)

    def restore():
        for s_, d_ in zip(pristine, work):
            d_.copy_(s_)
        flush.zero_()

    for _ in range(args.warmup):
        restore()
        run(work)
    torch.cuda.synchronize()
    if ws > 1:
        tdist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clk = ClockSampler(dev.index or 0).__enter__()
    time.sleep(0.2)
    torch.cuda.synchronize()
    n0 = idc.launch_count()
    t_wall0 = time.perf_counter()
    for k in range(args.steps):
        restore()
        evs[k][0].record(stream)
        run(work)
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall0
    launches = idc.launch_count() - n0
    samples = [e0.elapsed_time(e1) for e0, e1 in evs]
    # kernel pass: the same K calls again with the library's event profiler
    # bracketing every launch (kept out of the timed loop: its events
    # serialise the launches and add ~15% to a 0.1 ms call, profiles/r02/ab/)
    idc.profile_begin()
    for k in range(args.steps):
        restore()
        evs[k][0].record(stream)
        run(work)
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    prof = idc.profile_end()
    prof_step_ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / args.steps
    # the distributed path's NCCL exchanges (spans on the communicator's
    # stream, "A2A"): reported beside the kernels, not among them
    a2a = [r for r in prof if r["tag"] == "A2A"]
    prof = [r for r in prof if r["tag"] != "A2A"]
    a2a_rec = None
    if a2a:
        ms_a = sum(r["ms"] for r in a2a) / args.steps
        by = sum(r["units"] for r in a2a) / args.steps
        a2a_rec = {"ms_per_call": ms_a, "exchanges_per_call": sum(r["launches"] for r in a2a) / args.steps,
                   "bytes_sent_per_call": by, "gbs_per_rank": by / (ms_a / 1e3) / 1e9 if ms_a > 0 else None,
                   "how": "CUDA events around each grouped ncclSend/ncclRecv chunk on the communicator's stream "
                          "(overlapping phase B), this rank"}
    time.sleep(0.2)
    clk.__exit__()
    tot = torch.tensor([sum(samples)], dtype=torch.float64, device=dev)
    if ws > 1:
        tdist.all_reduce(tot, op=tdist.ReduceOp.MAX)
    total_ms = float(tot.item())
    sec = total_ms / 1e3 / args.steps
    pk = peaks()
    b, fl = part_model(p)
    convs = p["batch"] * (1 if dist3d else ws)        # strong (3D dist) or replicas (weak)
    ngpu_peak = ws
    t_b = b * convs / (pk["hbm_gbs"] * 1e9 * ngpu_peak)
    t_f = fl * convs / (pk["fp64_tflops"] * 1e12 * ngpu_peak)
    kt = kernel_table(p, prof, args.steps, pk, load_traffic(), prof_step_ms)
    # SURVEY 8(d) d.3 "measured" HBM GB/s: ncu DRAM bytes per unit of every
    # kernel class (profiles/traffic.json, one --set full capture each) x the
    # units of one call, over the call time
    dram_call = None
    if kt and all(k.get("traffic_per_launch") for k in kt):
        dram_call = sum(k["traffic_per_launch"] * k["launches_per_call"] for k in kt)
    out = dict(config=name, workload=p["desc"], kind=p["kind"], m=p["m"], batch=p["batch"],
               scaling="strong" if dist3d else "weak", ms_per_call=sec * 1e3, call_stats=timing_stats(samples),
               conv_per_s=convs / sec, hbm_gbs_alg=b * convs / sec / 1e9, fp64_tflops_alg=fl * convs / sec / 1e12,
               t_roof_ms=max(t_b, t_f) * 1e3, roofline_frac=max(t_b, t_f) / sec,
               bound="hbm" if t_b >= t_f else "alu", gpu_launches=launches, kernels=kt,
               roofline=dominant_roofline(kt, pk), clocks=clk.summary(), wall_s_timed_loop=t_wall,
               dram_bytes_per_call_ncu=dram_call, all_to_all=a2a_rec,
               hbm_gbs_measured=(dram_call * ws / sec / 1e9) if dram_call else None,   # all ranks
               kernel_pass={"ms_per_call": prof_step_ms, "steps": args.steps,
                            "how": "K more calls right after the timed loop, same restore + L2 flush, with "
                                   "idc_profile_begin/end events around every launch on its stream"})
    del work, flush
    if want_e2e and not dist3d:
        out["e2e"] = run_e2e(args, idc, torch, p, pristine, dev, ws, tdist)
    del pristine
    torch.cuda.empty_cache()
    return out


def run_e2e(args, idc, torch, p, pristine, dev, ws, tdist):
    """Same metric through the public API with HOST (pinned) buffers: every
    step copies its inputs host -> device, convolves, and copies the result
    device -> host, all inside the timed region.  Steps alternate between two
    CUDA streams with one pinned result buffer each (the public `out=`
    argument, so the pinned inputs stay as they were), so step k+1's
    host -> device copy overlaps step k's convolution and its device -> host
    copy (the two PCIe directions run concurrently); 1D kinds use one stream
    (the library's host path pipelines row chunks inside each call); timed
    with events from the first copy to the last result on the host."""
    host = [a.cpu().pin_memory() for a in pristine]
    adv = p["kind"] == "advection2d"
    ins = host[:1] if adv else host
    # 1D kinds: one stream -- idc_conv1d_host already overlaps the copies of
    # chunk c+1 and c-1 with the kernel of chunk c inside one call (on the
    # library's own copy streams, which concurrent calls would share)
    ns = 1 if p["kind"].endswith("1d") else 2
    outs = [torch.empty(host[0].shape, dtype=host[0].dtype, pin_memory=True) for _ in range(2)]
    streams = [torch.cuda.Stream(dev) for _ in range(ns)]
    bi = sum(a.numel() * 16 for a in ins)
    # small calls: more steps (>= 16, and >= ~2 GB of host -> device copies, so
    # that one host-side hiccup does not decide a region of a few milliseconds)
    steps = max(2, args.e2e_steps) if bi > 2e9 else max(16, args.e2e_steps, min(256, -(-int(2e9) // max(bi, 1))))
    bo = host[0].numel() * 16

    def step(k):
        s = streams[k % ns]
        if adv:                                          # device-only call: the copies around it
            with torch.cuda.stream(s):
                w = ins[0].to(dev, non_blocking=True)
                o = idc.advection2d(w, stream=s)
                outs[k % 2].copy_(o, non_blocking=True)
                del w, o
        else:
            getattr(idc, p["kind"])(*ins, stream=s, out=outs[k % 2])

    for k in range(2):                                   # warm-up: workspaces of both streams
        step(k)
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for s in streams:
        s.wait_event(e0)
    for k in range(steps):
        step(k)
    for s in streams:
        cur.wait_stream(s)
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    same = bool(torch.equal(outs[0], outs[1]))           # both buffers hold the same (deterministic) result
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if ws > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    convs = p["batch"] * ws * steps
    del host, outs, ins
    idc.free_workspaces()
    return {"value": convs / (float(t.item()) / 1e3), "unit": "conv/s", "h2d_bytes_per_step": bi,
            "d2h_bytes_per_step": bo, "steps": steps, "streams": ns, "results_identical": same,
            "how": "idconv.<kind>(pinned host inputs, stream=s_(k mod streams), out=pinned host buffer (k mod 2)); "
                   "H2D + convolution + D2H of every step inside one event-timed region"}


def run_ours(args):
    import torch
    import torch.distributed as tdist
    from paper_1008_1366_b200 import idconv as idc

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")            # communicator lines (NVLS, nranks) on stderr
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        tdist.init_process_group("nccl", device_id=dev)
        comm = idc.Comm()
    parts_names = [x for x in args.parts.split(",") if x] if args.parts else []
    parts_names = [x for x in parts_names if x != args.workload]
    parts = []
    for name in parts_names:
        parts.append(measure(idc, torch, tdist, name, args, rank, ws, dev, comm=comm,
                             want_e2e=(not args.no_e2e and ws == 1)))
    head = measure(idc, torch, tdist, args.workload, args, rank, ws, dev, comm=comm, want_e2e=not args.no_e2e)
    if comm is not None:
        comm.close()
    out = None
    if rank == 0:
        hp = CONFIGS[args.workload]
        out = {
            "metric": METRIC, "value": head["conv_per_s"], "unit": "conv/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_call"], "higher_is_better": True,
            "scaling": head["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": head["workload"], "kind": hp["kind"], "m": hp["m"], "batch": hp["batch"],
                       "parallelism": (f"x-slabs{ws} (NCCL all-to-all)" if head["scaling"] == "strong" and ws > 1
                                       else f"replicas{ws}"),
                       "l2": "inputs (> L2) restored from pristine device copies and a 256 MB buffer written "
                             "(L2 flush) before every timed call",
                       "seed": synthgen.SEED},
            "roofline": head["roofline"],
            "call_roofline": {"bound": head["bound"], "frac": head["roofline_frac"], "t_roof_ms": head["t_roof_ms"],
                              "hbm_gbs_alg": head["hbm_gbs_alg"], "fp64_tflops_alg": head["fp64_tflops_alg"],
                              "dram_bytes_per_call_ncu": head["dram_bytes_per_call_ncu"],
                              "hbm_gbs_measured": head["hbm_gbs_measured"]},
            "e2e": head.get("e2e"), "gpu_launches": head["gpu_launches"], "clocks": head["clocks"],
            "call_stats": head["call_stats"], "kernels": head["kernels"], "kernel_pass": head["kernel_pass"],
            "all_to_all": head["all_to_all"],
            "wall_s_timed_loop": head["wall_s_timed_loop"], "parts": parts,
        }
        if ws > 1:
            out["nccl"] = {"backend": "nccl", "nranks": ws, "version": ".".join(map(str, torch.cuda.nccl.version())),
                           "debug": os.environ.get("NCCL_DEBUG")}
    if ws == 1 and rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.workload, args.cpu_budget)
        for pt in parts:
            pt["cpu_baseline"] = cpu_baseline(pt["config"], args.cpu_budget_part)
    elif out is not None:
        out["cpu_baseline"] = None
    if ws > 1:
        tdist.barrier()
        tdist.destroy_process_group()
    return out


# ----------------------------------------------------------- oracle (CPU) --

def _oracle_inputs(p):
    kind = p["kind"]
    if kind in ("cconv2d",):
        f, g = synthgen.cconv2d_inputs(*p["m"], 1)
        return [f[0], g[0]]
    if kind == "hconv2d":
        return list(synthgen.hconv2d_inputs(*p["m"]))
    if kind == "advection2d":                  # the vorticity w (one array)
        return [synthgen.hconv2d_inputs(*p["m"], roles=(0,))[0]]
    if kind == "cconv3d":
        return list(synthgen.cconv3d_inputs(*p["m"]))
    if kind == "hconv3d":
        return list(synthgen.hconv3d_inputs(*p["m"]))
    raise ValueError(kind)


class OracleSampler:
    """The CPU oracle (direct sums, oracle/direct.c) on bounded samples of a
    config: 1D kinds a number of whole rows; 2D/3D kinds random output points
    (3D: random (x, y) lines with several z each), extrapolated to whole
    convolutions from the measured time per output point."""

    def __init__(self, name):
        from oracle import direct
        self.d = direct
        self.p = CONFIGS[name]
        self.name = name
        self.rs = np.random.default_rng(1008)
        kind = self.p["kind"]
        if kind.endswith("1d") or kind == "tconv2d":
            self.arrs = None
        else:
            self.arrs = _oracle_inputs(self.p)

    def sample(self, budget_s):
        """Run the oracle for about budget_s seconds; returns (convs, secs, desc)."""
        p, kind, d = self.p, self.p["kind"], self.d
        t_end = time.perf_counter() + budget_s
        secs, done = 0.0, 0
        if kind.endswith("1d"):
            fn = {"cconv1d": d.cconv1d, "hconv1d": d.hconv1d, "tconv1d": d.tconv1d}[kind]
            while True:
                rows = [self.rs.integers(0, p["batch"])]
                arrs = [np.stack([synthgen.uniform_complex(p["m"], synthgen.array_id(r, b)) for b in rows])
                        for r in range(p["narr"])]
                if kind != "cconv1d":
                    for a in arrs:
                        a[:, 0] = a[:, 0].real
                t0 = time.perf_counter()
                fn(*arrs)
                secs += time.perf_counter() - t0
                done += 1
                if time.perf_counter() > t_end:
                    break
            return done, secs, f"{done} whole rows of {p['batch']} ({kind}, m={p['m']})"
        if kind == "tconv2d":
            return self._sample_tconv2d(budget_s)
        f, g = (self.arrs + [None])[:2]
        npts = 0
        while True:
            if kind == "advection2d":
                idx = self.rs.choice(f.size, 2, replace=False)
                t0 = time.perf_counter()
                from oracle import application
                application.euler_sum_at(f, idx)
            elif kind == "cconv2d":
                idx = self.rs.choice(f.size, 4, replace=False)
                t0 = time.perf_counter()
                d.cconv_nd_at(f, g, idx)
            elif kind == "hconv2d":
                idx = self.rs.choice(f.size, 4, replace=False)
                t0 = time.perf_counter()
                d.hconv2d_at(f, g, idx)
            elif kind == "cconv3d":
                idx = self.rs.choice(f.size, 4, replace=False)
                t0 = time.perf_counter()
                d.cconv3d_at_large(f, g, idx)
            else:   # hconv3d: one random (x, y) line, 4 random z on it
                i, j = self.rs.integers(0, f.shape[0]), self.rs.integers(0, f.shape[1])
                kz = self.rs.choice(f.shape[2], 4, replace=False)
                idx = np.ravel_multi_index((np.full(4, i), np.full(4, j), kz), f.shape)
                t0 = time.perf_counter()
                d.hconv3d_at_lines(f, g, idx)
            secs += time.perf_counter() - t0
            npts += len(idx)
            if time.perf_counter() > t_end:
                break
        per_pt = secs / npts
        convs = secs / (per_pt * outputs_per_conv(p))   # whole convolutions' worth of oracle time
        return convs, secs, (f"{npts} random outputs of the {'x'.join(map(str, shape_of(p)))} output "
                             f"({kind}), direct sums, {per_pt * 1e3:.1f} ms per output; "
                             f"EXTRAPOLATED to {outputs_per_conv(p)} outputs per convolution")


    def _sample_tconv2d(self, budget_s):
        """One output of the 2D ternary sum costs ~(2m)^4 products (2.8e14 at
        m = 2048), so not one output of the real size fits the budget: the
        oracle (ternary2d.direct, two stages of direct 2D convolution) runs
        whole at mx = my = ms and the time is scaled by the operation count of
        the two stages, ((2m-1)^2 (2m-1)^2 + (4m-3)^2 (2m-1)^2), to the
        config's m.  EXTRAPOLATED, and labelled so."""
        from oracle import ternary2d
        mx, my = self.p["m"]
        ms = 16

        def cost(a, b):
            return (2 * a - 1) ** 2 * (2 * b - 1) ** 2 + (4 * a - 3) * (4 * b - 3) * (2 * a - 1) * (2 * b - 1)

        f, g, h = synthgen.hconv2d_inputs(ms, ms, roles=(0, 1, 2))
        arrs = [np.concatenate([np.zeros((1, ms), np.complex128), a]) for a in (f, g, h)]
        t_end = time.perf_counter() + budget_s
        secs, done = 0.0, 0
        while True:
            t0 = time.perf_counter()
            ternary2d.direct(*arrs)
            secs += time.perf_counter() - t0
            done += 1
            if time.perf_counter() > t_end:
                break
        scale = cost(mx, my) / cost(ms, ms)
        convs = done / scale
        return convs, secs, (f"{done} whole tconv2d at mx = my = {ms} (ternary2d.direct, scipy direct 2D "
                             f"convolution, {secs / done * 1e3:.2f} ms each); EXTRAPOLATED to mx = {mx}, my = {my} "
                             f"by the two stages' product count (x{scale:.3g})")


def cpu_baseline(name, budget):
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    s = OracleSampler(name)
    convs, secs, desc = s.sample(budget)
    if CONFIGS[name]["kind"] in ("advection2d", "tconv2d"):    # numpy / scipy sums, one thread
        return {"value": convs / secs, "unit": "conv/s", "cores": 1, "kind": "oracle",
                "sample": desc + " -- oracle/__init__.py (numpy / scipy sums)"}
    return {"value": convs / secs, "unit": "conv/s", "cores": threads, "kind": "oracle",
            "sample": desc + " -- oracle/direct.c (TwoProd + Neumaier / Dot2 compensated, OpenMP)"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    p = CONFIGS[args.workload]
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    s = OracleSampler(args.workload)
    budget = max(1.0, args.cpu_budget / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        s.sample(budget)
    convs, secs, desc = 0.0, 0.0, ""
    for _ in range(args.steps):
        c, t, desc = s.sample(budget)
        convs += c
        secs += t
    value = convs / secs
    return {"metric": METRIC, "value": value, "unit": "conv/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": p["desc"], "kind": p["kind"], "m": p["m"], "batch": p["batch"],
                       "parallelism": "host cores", "seed": synthgen.SEED},
            "cpu_baseline": {"value": value, "unit": "conv/s", "cores": threads, "kind": "oracle",
                             "sample": desc + " per step"},
            "e2e": {"value": value, "unit": "conv/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# --------------------------------------------------- multi-process launch --

def spawn(args, argv):
    """--gpus N launched directly (no torchrun env): re-launch this script
    under torch.distributed.run with N local ranks on 127.0.0.1."""
    import random
    port = 29500 + random.randrange(0, 2000)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


def dry_run(args):
    """Rendezvous check without GPUs: every rank joins a gloo group and
    reports itself; rank 0 prints the plan as one JSON line."""
    import torch
    import torch.distributed as tdist
    ws, rank, _ = dist_env()
    if ws > 1:
        tdist.init_process_group("gloo")
        t = torch.zeros(ws, dtype=torch.int64)
        t[rank] = os.getpid()
        tdist.all_reduce(t)
        pids = t.tolist()
        tdist.destroy_process_group()
    else:
        pids = [os.getpid()]
    if rank == 0:
        return {"dry_run": True, "n_gpus": args.gpus, "world_size": ws, "rank_pids": pids,
                "headline": args.workload, "parts": args.parts,
                "plan": ("3D configs slab-sharded over the ranks (idc_*conv3d_dist), 1D/2D replicas"
                         if ws > 1 else "single GPU")}
    return None


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="idconv", choices=["idconv", "reference"])
    ap.add_argument("--workload", default=HEADLINE, choices=sorted(CONFIGS), help="headline config")
    ap.add_argument("--parts", default=DEFAULT_PARTS, help="comma-separated configs measured besides the headline")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of oracle CPU work (headline)")
    ap.add_argument("--cpu-budget-part", type=float, default=3.0, help="seconds of oracle CPU work per part")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="spawn/rendezvous check only (no GPU)")
    args = ap.parse_args(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args, argv))
    if args.dry_run:
        out = dry_run(args)
    elif args.impl == "reference":
        out = run_reference(args)
    else:
        if args.warmup < 3:
            print("warning: the contract asks for >= 3 warm-up steps", file=sys.stderr)
        out = run_ours(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
