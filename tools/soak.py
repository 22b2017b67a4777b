"""Soak test: repeated hconv3d (C5b) calls with inputs restored before each,
per-call CUDA-event times and nvidia-smi clocks / power / throttle reasons
sampled alongside (finds intermittent slowdowns)."""
import json
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1008_1366_b200 import idconv

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 90
kind = sys.argv[2] if len(sys.argv) > 2 else "hconv3d"
shape = (1023, 1023, 512) if kind == "hconv3d" else (512, 512, 512)
rows = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,power.draw,temperature.gpu,"
                         "clocks_event_reasons.active", "--format=csv,noheader", "-lms", "500"],
                        stdout=subprocess.PIPE, text=True)
threading.Thread(target=lambda: [rows.append(l.strip()) for l in proc.stdout], daemon=True).start()
src = [torch.empty(shape, dtype=torch.complex128, device="cuda") for _ in range(2)]
for i, a in enumerate(src):
    idconv.fill_uniform(a, i, 1)
    a /= 1e3
work = [torch.empty_like(a) for a in src]
t0 = time.time()
times = []
while time.time() - t0 < secs:
    for s_, d_ in zip(src, work):
        d_.copy_(s_)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    getattr(idconv, kind)(*work)
    e1.record()
    torch.cuda.synchronize()
    times.append((round(time.time() - t0, 2), round(e0.elapsed_time(e1), 2)))
proc.terminate()
print(json.dumps({"kind": kind, "n": len(times), "min": min(t for _, t in times), "max": max(t for _, t in times)}))
for t, ms in times[:: max(1, len(times) // 60)]:
    print(t, ms)
print("--- smi")
for r in rows[:: max(1, len(rows) // 60)]:
    print(r)
