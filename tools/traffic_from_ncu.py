"""DRAM bytes per unit (row or pencil column) of a kernel class from one
`ncu --set full` capture, merged into profiles/traffic.json (read by
bench.py for the roofline "traffic" field: bytes per unit x units per launch).

usage: python tools/traffic_from_ncu.py <report.ncu-rep | raw.csv> <tag:n> <units in that launch> [note]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, key, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
note = sys.argv[4] if len(sys.argv) > 4 else ""
if rep.endswith(".csv"):                       # `ncu -i ... --page raw --csv` output saved on the GPU box
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def get(k):
    return float(v[h.index(k)].replace(",", "")) * scale.get(u[h.index(k)], 1.0)


tot = get("dram__bytes_read.sum") + get("dram__bytes_write.sum")
path = os.path.join(ROOT, "profiles", "traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d[key] = tot / units
meta = d.setdefault("_source", {})
meta[key] = f"{os.path.basename(rep)}: {tot:.4g} B DRAM over {units:.0f} units{(' -- ' + note) if note else ''}"
json.dump(d, open(path, "w"), indent=1, sort_keys=True)
print(key, tot / units)
