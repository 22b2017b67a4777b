"""p/q implicit padding (NEXT-3) timing: rows of L = p*m modes, implicit q*m
padding vs the explicitly padded cuFFT convolution (comparison only) and the
power-of-two implicit cconv1d at the next length."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1008_1366_b200 import idconv
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import cufft_explicit as ex


def timed(fn, prep, reps=5):
    best = None
    for _ in range(reps):
        prep()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        t = a.elapsed_time(b)
        best = t if best is None else min(best, t)
    return best


rows = []
for (p, q, m, B) in [(3, 7, 1024, 8192), (3, 6, 1024, 8192), (1, 2, 1024, 24576), (2, 5, 512, 16384)]:
    L = p * m
    f0 = torch.empty((B, L), dtype=torch.complex128, device="cuda"); g0 = torch.empty_like(f0)
    idconv.fill_uniform(f0, 0, 1); idconv.fill_uniform(g0, 1, 1)
    f, g = f0.clone(), g0.clone()
    def prep():
        f.copy_(f0); g.copy_(g0)
    t_pq = timed(lambda: idconv.cconv1d_pq(f, g, p, q), prep)
    ref = ex.cconv1d(f0, g0)
    idconv.cconv1d_pq(f, g, p, q) if False else None
    prep(); idconv.cconv1d_pq(f, g, p, q); torch.cuda.synchronize()
    err = float(torch.linalg.vector_norm(f - ref) / torch.linalg.vector_norm(ref))
    t_ex = timed(lambda: ex.cconv1d(f0, g0), lambda: None)
    row = dict(p=p, q=q, m=m, L=L, batch=B, implicit_pq_ms=t_pq, explicit_cufft_ms=t_ex,
               conv_per_s=B / (t_pq / 1e3), hbm_gbs_alg=3 * 16 * L * B / (t_pq / 1e3) / 1e9, rel_l2_vs_explicit=err)
    print(json.dumps(row), flush=True)
    rows.append(row)
