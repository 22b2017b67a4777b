"""Host enqueue time vs device time of one ND call (is the call launch-bound?)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1008_1366_b200 import idconv
kind = sys.argv[1]; shape = tuple(int(x) for x in sys.argv[2].split(","))
f = torch.empty(shape, dtype=torch.complex128, device="cuda"); g = torch.empty_like(f)
idconv.fill_uniform(f, 0, 1); idconv.fill_uniform(g, 1, 1)
fn = getattr(idconv, kind)
for r in range(3):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(); fn(f, g); e1.record(); t1 = time.perf_counter()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"{kind} {shape}: enqueue {1e3*(t1-t0):.2f} ms, device {e0.elapsed_time(e1):.2f} ms, wall {1e3*(t2-t0):.2f} ms")
