"""Print the key ncu metrics, stall mix and per-opcode stall attribution of
an .ncu-rep (reads `ncu -i ... --page raw/source --csv`)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
        "smsp__sass_inst_executed_op_shared_st.sum", "smsp__sass_inst_executed_op_local_ld.sum",
        "smsp__sass_inst_executed_op_global_ld.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for w in want:
    if w in h:
        print(f"{w} = {v[h.index(w)]} {u[h.index(w)]}")
st = [(h[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v[i].replace(",", "") or 0)) for i in range(len(h))
      if h[i].startswith("smsp__pcsamp_warps_issue_stalled") and not h[i].endswith("not_issued")]
tot = sum(b for a, b in st) or 1
st.sort(key=lambda x: -x[1])
print("stalls: " + " ".join(f"{a}:{100 * b / tot:.0f}%" for a, b in st[:10]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
hh = srows[1]
iS = hh.index("Source")
iW = hh.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in hh else None
iSt = [j for j, x in enumerate(hh) if x.startswith("stall_") and "Not Issued" not in x]
iE = hh.index("Instructions Executed")
agg, ins, wf = collections.Counter(), collections.Counter(), collections.Counter()
for r in srows[2:]:
    parts = r[iS].split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") else parts[0]
    op = op.split(".")[0]
    try:
        ins[op] += float(r[iE] or 0)
        if iW is not None:
            wf[op] += float(r[iW] or 0)
    except ValueError:
        pass
    for j in iSt:
        try:
            agg[(op, hh[j])] += float(r[j] or 0)
        except ValueError:
            pass
tot = sum(agg.values()) or 1
print("top (opcode, stall):", ", ".join(f"{o}/{s[6:]}:{100 * x / tot:.1f}%" for (o, s), x in agg.most_common(14)))
print("warp-instructions by opcode:", ", ".join(f"{o}:{x / 1e6:.1f}M" for o, x in ins.most_common(14)))
if iW is not None:
    print("shared wavefronts by opcode:", ", ".join(f"{o}:{x / 1e6:.1f}M" for o, x in wf.most_common(6)))
