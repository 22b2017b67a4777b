"""Upper bound of what L2-resident slab groups could buy:
the slab-phase kernels of config 5b (K7/K8 along y on 1023-row columns, K3 on
512-point z rows) timed on problems that fit in L2 (back-to-back calls, no
flush) against the same per-unit work streaming from HBM (large problems, or
L2 flushed between calls).

usage: python tools/l2_potential.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1008_1366_b200 import idconv


def timed(fn, arrs, calls, reps=5):
    """median over reps of (calls back-to-back calls between two events) / calls;
    no flush, so an L2-sized problem stays resident from call to call (inputs
    of magnitude ~1e-3: the repeated in-place convolutions stay finite)"""
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(calls):
            fn(*arrs)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / calls)
    ts.sort()
    return ts[len(ts) // 2]


def inputs(shape, n=2):
    arrs = [torch.empty(shape, dtype=torch.complex128, device="cuda") for _ in range(n)]
    for i, x in enumerate(arrs):
        idconv.fill_uniform(x, i, 1)
        x.mul_(1e-3)
    return arrs


def main():
    # K3 rows, m = 512: 4096 rows (2 x 32 MB, L2-resident) vs 65536 rows (2 x 512 MB, streaming)
    for B in (4096, 65536):
        ms = timed(idconv.hconv1d, inputs((B, 512)), 20)
        print(f"hconv1d m=512 B={B}: {ms:.4f} ms per call, {ms * 1e6 / B:.2f} ns/row")
    # one C5b slab as a 2D hconv (K7 along y, K3 on the 1536 z rows, K8): 2 x 8.4 MB, L2-resident
    ms = timed(idconv.hconv2d, inputs((1023, 512)), 50)
    print(f"hconv2d 1023x512 (one C5b slab, L2-resident, back to back): {ms:.4f} ms per slab, x 1535 slabs = {ms * 1535:.1f} ms")
    ms = timed(idconv.hconv3d, inputs((1023, 1023, 512)), 1, reps=3)
    print(f"hconv3d 1023^2 x 512: {ms:.3f} ms per call")


if __name__ == "__main__":
    main()
