"""One call of an ND kind at a config size (for ncu launch lists / timing)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1008_1366_b200 import idconv
ap = argparse.ArgumentParser()
ap.add_argument("kind")
ap.add_argument("shape")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
shape = tuple(int(x) for x in a.shape.split(","))
narr = 3 if a.kind == "tconv2d" else 2
arrs = [torch.empty(shape, dtype=torch.complex128, device="cuda") for _ in range(narr)]
for i, x in enumerate(arrs):
    idconv.fill_uniform(x, i, 1)
fn = getattr(idconv, a.kind)
for r in range(a.reps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); fn(*arrs); e1.record(); torch.cuda.synchronize()
    print(a.kind, shape, "%.3f ms" % e0.elapsed_time(e1))
