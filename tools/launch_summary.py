"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
skip = sys.argv[2] if len(sys.argv) > 2 else "k_fill_uniform"
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= iv or r[im] != "gpu__time_duration.sum" or skip in r[ik]:
        continue
    name = r[ik].split("(")[0].replace("void ", "")[:70]
    agg[name][0] += 1
    agg[name][1] += float(r[iv].replace(",", ""))
tot = sum(v for c, v in agg.values())
print(f"total {tot/1e6:.3f} ms over {sum(c for c, v in agg.values())} launches")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:15]:
    print(f"{n:70s} n={c:6d} {v/1e6:9.3f} ms {100*v/tot:5.1f}%  avg {v/c/1e3:8.1f} us")
