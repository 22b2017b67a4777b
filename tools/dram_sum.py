"""Sum ncu DRAM bytes / time over the hot-path launches of a launch-list CSV."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ik, im, iu, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
tot = defaultdict(float)
per = defaultdict(lambda: defaultdict(float))
for r in rows[hi + 1:]:
    if len(r) <= iv or "idc::" not in r[ik]:
        continue
    v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
    tot[r[im]] += v
    per[r[ik].split("(")[0].replace("void ", "")][r[im]] += v
rd, wr, t = tot["dram__bytes_read.sum"], tot["dram__bytes_write.sum"], tot["gpu__time_duration.sum"]
print(f"{sys.argv[1]}: DRAM read {rd / 1e9:.2f} GB + write {wr / 1e9:.2f} GB = {(rd + wr) / 1e9:.2f} GB over "
      f"{t * 1e3:.2f} ms of kernel time (serialised)")
for k, d in sorted(per.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    print(f"  {k:40s} {(d['dram__bytes_read.sum'] + d['dram__bytes_write.sum']) / 1e9:8.2f} GB  "
          f"{d['gpu__time_duration.sum'] * 1e3:8.2f} ms")
