"""Run one row-kernel launch configuration a few times (for ncu / timing)."""
import argparse
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1008_1366_b200 import idconv

ap = argparse.ArgumentParser()
ap.add_argument("kind")
ap.add_argument("m", type=int)
ap.add_argument("batch", type=int)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n = 3 if a.kind == "tconv1d" else 2
arrs = [torch.empty((a.batch, a.m), dtype=torch.complex128, device="cuda") for _ in range(n)]
for i, x in enumerate(arrs):
    idconv.fill_uniform(x, i, 1)
fn = getattr(idconv, a.kind)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for r in range(a.reps):
    ev[0].record()
    fn(*arrs)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    print(f"{a.kind} m={a.m} B={a.batch}: {ms:.3f} ms, {ms*1e6/a.batch:.1f} ns/conv")
