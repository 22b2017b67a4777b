"""Copy one GPU evidence session (tools/gpu_round.sh <tag>) from gpurun_out/
into profiles/: bench lines, ncu launch list + summary, ncu --set full
metric summaries of the dominant kernels and traffic.json (DRAM bytes per
launch, read by bench.py for the roofline "traffic" field)."""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = os.path.join(ROOT, "gpurun_out")
dst = os.environ.get("PROFILES_OUT", os.path.join(ROOT, "profiles"))   # run on the GPU box: a gpurun_out/ subdir
os.makedirs(dst, exist_ok=True)

for w in ["c2", "c1", "c3a", "c3b", "c4", "c4adv", "c4t", "c5a", "c5b", "ref"]:
    p = os.path.join(src, f"{tag}_bench_{w}.json")
    if os.path.exists(p):
        shutil.copy(p, os.path.join(dst, f"{tag}_bench_{w}.json"))
for f in [f"{tag}_launches_c2.csv", f"{tag}_launches_c2_summary.txt", f"{tag}_smi.txt", f"{tag}_cufft_compare.json",
          f"{tag}_pcie.json"]:
    if os.path.exists(os.path.join(src, f)):
        shutil.copy(os.path.join(src, f), os.path.join(dst, f))

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "smsp__inst_executed.sum", "smsp__sass_inst_executed_op_local_ld.sum",
           "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
           "smsp__sass_inst_executed_op_global_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "sm__cycles_elapsed.avg.per_second"]
UNIT = {"gpu__time_duration.sum": 1e3, "dram__bytes_read.sum": 1e6, "dram__bytes_write.sum": 1e6}
CASES = [("tconv", "tconv1d", 4096, 4096), ("hconv", "hconv1d", 4096, 4096), ("cconv", "cconv1d", 1024, 32768)]
traffic = {}
lines = [f"# {tag}: ncu --set full captures of the dominant row kernels", "",
         "Command: `ncu --set full --import-source on --clock-control none -k regex:_rows -c 1 "
         "python tools/prof_rows.py <kind> <m> <batch>` (tools/prof_one.sh; one launch, cold cache, replayed).", ""]
for short, kind, m, batch in CASES:
    rep = os.path.join(src, f"{tag}_prof_{short}.ncu-rep")
    if not os.path.exists(rep):
        continue
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    get = lambda k: float(v[h.index(k)].replace(",", "")) if k in h else None

    def to_base(k):
        x = get(k)
        u = units[h.index(k)] if k in h else ""
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "msecond": 1e-3, "usecond": 1e-6,
                 "nsecond": 1e-9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0}.get(u, 1.0)
        return x * scale if x is not None else None
    rd, wr, dur = to_base("dram__bytes_read.sum"), to_base("dram__bytes_write.sum"), to_base("gpu__time_duration.sum")
    traffic[f"{kind}:{m}"] = rd + wr
    alg = (4 if kind == "tconv1d" else 3) * 16 * m * batch
    stalls = [(h[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v[i].replace(",", "") or 0))
              for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled")
              and not h[i].endswith("not_issued") and v[i].replace(",", "").replace(".", "").isdigit()]
    tot = sum(b for a, b in stalls) or 1
    stalls.sort(key=lambda x: -x[1])
    lines += [f"## {kind} m={m}, batch {batch} (`{tag}_prof_{short}.ncu-rep`, in gpurun_out/)", "",
              f"* duration {dur * 1e3:.3f} ms (ncu replay, cold cache)",
              f"* DRAM read {rd / 1e6:.1f} MB + write {wr / 1e6:.1f} MB = {(rd + wr) / 1e6:.1f} MB "
              f"vs algorithmic {alg / 1e6:.1f} MB ({(rd + wr) / alg:.2f}x)"]
    for k in METRICS:
        if k in h:
            lines.append(f"* `{k}` = {v[h.index(k)]} {units[h.index(k)]}")
    lines.append("* stall mix (pc sampling): " + ", ".join(f"{a} {100 * b / tot:.0f}%" for a, b in stalls[:9]))
    lines.append("")
with open(os.path.join(dst, f"{tag}_ncu_full_summary.md"), "w") as fh:
    fh.write("\n".join(lines) + "\n")
with open(os.path.join(dst, "traffic.json"), "w") as fh:
    json.dump(traffic, fh, indent=1)

# ---- 2D / 3D kernels (tools/prof_nd_full.sh <tag>nd) ----
ND = [("c4_rows", "K3 hconv rows3<2048>, C4 (6143 rows, both x-streams)"),
      ("c4_k7", "K7 fft0padBackward<2048>, C4 x pass"), ("c4_k8", "K8 fft0padForward<2048>, C4 x pass"),
      ("c5a_k5x", "K5 fftpadBackward<512>, C5a x pass (all (y,z) columns)"),
      ("c5a_rows", "K2 cconv rows2<512>, C5a first slab group"), ("c5b_k7x", "K7 fft0padBackward<512>, C5b x pass"),
      ("c5b_rows", "K3 hconv rows3<512>, C5b first slab group"),
      ("c4t_k5", "K5 fftpadBackward<4096>, C4t x pass (f, g)"), ("c4t_rows", "K4 tconv rows3<2048>, C4t"),
      ("c3a_k5", "K5 fftpadBackward<1024>, C3a x pass"), ("c3a_rows", "K2 cconv rows2<1024>, C3a")]
nd = [f"# {tag}: ncu --set full captures of the dominant 2D / 3D kernels", "",
      "Command: `tools/prof_nd_full.sh` (first launch of each kernel in one call of the config, `ncu --set full "
      "--import-source on --clock-control none -k regex:<kernel> -c 1`, cold cache, replayed). Reports stay in "
      "gpurun_out/ (too large to commit).", "",
      "| kernel | time | DRAM read + write | DRAM GB/s | fp64 pipe | L1/shared | issue | warps | regs | local ld | "
      "top stalls |", "|---|---|---|---|---|---|---|---|---|---|---|"]
for short, label in ND:
    rep = os.path.join(src, f"{tag}nd_{short}.ncu-rep")
    if not os.path.exists(rep):
        continue
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    sc = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "msecond": 1e-3, "usecond": 1e-6,
          "nsecond": 1e-9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0}
    val = lambda k: float(v[h.index(k)].replace(",", "")) * sc.get(units[h.index(k)], 1.0)
    raw = lambda k: float(v[h.index(k)].replace(",", ""))
    dur, rd, wr = val("gpu__time_duration.sum"), val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    stalls = [(h[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v[i].replace(",", "") or 0))
              for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled")
              and not h[i].endswith("not_issued") and v[i].replace(",", "").replace(".", "").isdigit()]
    tot = sum(b for a, b in stalls) or 1
    stalls.sort(key=lambda x: -x[1])
    nd.append(f"| {label} | {dur * 1e6:.1f} us | {rd / 1e6:.0f} + {wr / 1e6:.0f} MB | {(rd + wr) / dur / 1e9:.0f} | "
              f"{raw('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.0f}% | "
              f"{raw('l1tex__throughput.avg.pct_of_peak_sustained_active'):.0f}% | "
              f"{raw('smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f}% | "
              f"{raw('sm__warps_active.avg.pct_of_peak_sustained_active'):.0f}% | "
              f"{raw('launch__registers_per_thread'):.0f} | {raw('smsp__sass_inst_executed_op_local_ld.sum'):.0f} | "
              + ", ".join(f"{a} {100 * b / tot:.0f}%" for a, b in stalls[:3]) + " |")
if len(nd) == 6 + len(ND):   # only a complete capture set replaces the committed summary
    with open(os.path.join(dst, f"{tag}_ncu_nd_summary.md"), "w") as fh:
        fh.write("\n".join(nd) + "\n")
print("wrote", dst, sorted(os.listdir(dst)))
