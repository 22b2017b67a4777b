"""DRAM traffic of every kernel class of the 2D configs (the pencil and
dot-product kernels that profiles/traffic.json lacked), for bench.py's
`traffic` fields.

On the GPU box:
  python tools/traffic_sweep.py units > gpurun_out/traffic_units.json
  ncu --set full --clock-control none -k regex:'^k_|::k_' -o gpurun_out/traffic_sweep \
      python tools/traffic_sweep.py run
  ncu -i gpurun_out/traffic_sweep.ncu-rep --page raw --csv > gpurun_out/traffic_sweep.raw.csv
Here:
  python tools/traffic_sweep.py merge gpurun_out/traffic_units.json gpurun_out/traffic_sweep.raw.csv

`run` makes one call per config (inputs from bench.make_inputs, i.e. the
library's k_fill_uniform launches, which also separate the configs in the
launch list); `units` makes the same calls with the library's profiler on and
prints the units (rows or pencil columns) of each kernel class; `merge` sums
ncu's dram__bytes_read + dram__bytes_write per class and config and writes
bytes per unit into profiles/traffic.json under "<config>:<tag>:<n>"."""
import csv
import io
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CONFIGS = ["c3a", "c3b", "c4", "c4adv", "c4t"]
TAGS = {"k_pad_bwd_tma": "K5", "k_pad_fwd_tma": "K6", "k_pad0_bwd_tma": "K7", "k_pad0_fwd_tma": "K8",
        "k_cconv_rows2": "K2", "k_hconv_rows3": "K3", "k_tconv_rows3": "K4", "k_hconv_dot_rows": "K3d",
        "k_advection2d_inputs": "Kadv"}


def calls(profile):
    import torch

    import bench
    from paper_1008_1366_b200 import idconv as idc
    dev = torch.device("cuda", 0)
    out = {}
    for name in CONFIGS:
        p = dict(bench.CONFIGS[name], name=name)
        arrs = bench.make_inputs(idc, torch, p, 0, dev)
        bench.call(idc, p, arrs)                    # warm-up (tables, workspace)
        arrs = bench.make_inputs(idc, torch, p, 0, dev)
        torch.cuda.synchronize()
        if profile:
            idc.profile_begin()
        bench.call(idc, p, arrs)
        torch.cuda.synchronize()
        if profile:
            out[name] = idc.profile_end()
        del arrs
        torch.cuda.empty_cache()
    return out


def merge(units_path, raw_path):
    units = json.load(open(units_path))
    rows = list(csv.reader(io.StringIO(open(raw_path).read())))
    h, u = rows[0], rows[1]
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    kn = h.index("Kernel Name")

    def val(r, k):
        return float(r[h.index(k)].replace(",", "")) * scale.get(u[h.index(k)], 1.0)

    # launch list -> calls: each config makes its warm-up call, then the timed
    # call, both preceded by the fill kernels of its inputs
    seq = []
    for r in rows[2:]:
        name = r[kn]
        base = re.search(r"\b(k_[a-z0-9_]+)", name)
        base = base.group(1) if base else name
        if base == "k_fill_uniform":
            if not seq or seq[-1]:
                seq.append([])
            continue
        n = re.search(r"<\(?(?:int)?\)?(\d+)", name)
        seq[-1].append((TAGS.get(base, base), int(n.group(1)) if n else 0,
                        val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")))
    seq = [s for s in seq if s]
    assert len(seq) == 2 * len(CONFIGS), f"{len(seq)} call groups in the launch list"
    path = os.path.join(ROOT, "profiles", "traffic.json")
    d = json.load(open(path))
    meta = d.setdefault("_source", {})
    for i, name in enumerate(CONFIGS):
        launches = seq[2 * i + 1]                  # the second call of the config
        per = {}
        for tag, n, b in launches:
            per[(tag, n)] = per.get((tag, n), 0.0) + b
        for rec in units[name]:
            key = (rec["tag"], rec["n"])
            if key not in per:
                key = (rec["tag"], 0)          # kernels without a size template (Kadv)
            if key not in per:
                continue
            k = f"{name}:{rec['tag']}:{rec['n']}"
            d[k] = per[key] / rec["units"]
            meta[k] = (f"{os.path.basename(raw_path)}: {per[key]:.4g} B DRAM over {rec['units']} units "
                       f"({rec['launches']} launch(es)) -- tools/traffic_sweep.py, config {name}")
            print(k, d[k])
    json.dump(d, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "units":
        print(json.dumps(calls(True)))
    elif mode == "run":
        calls(False)
    else:
        merge(sys.argv[2], sys.argv[3])
