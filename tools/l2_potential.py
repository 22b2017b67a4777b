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


def timed(fn, arrs, reps, flush=None):
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(*arrs)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    # K3 rows, m = 512: 2048 rows (2 x 16 MB, L2-resident) vs 65536 rows (2 x 512 MB)
    for B, fl in ((2048, False), (2048, True), (65536, False)):
        arrs = [torch.empty((B, 512), dtype=torch.complex128, device="cuda") for _ in range(2)]
        for i, x in enumerate(arrs):
            idconv.fill_uniform(x, i, 1)
        ms = timed(idconv.hconv1d, arrs, 21, flush if fl else None)
        print(f"hconv1d m=512 B={B} {'flushed' if fl else 'no flush'}: {ms:.4f} ms, {ms * 1e6 / B:.2f} ns/row")
    # one C5b slab as a 2D hconv (K7 along y, K3 on z rows, K8): 2 x 8.4 MB
    for fl in (False, True):
        arrs = [torch.empty((1023, 512), dtype=torch.complex128, device="cuda") for _ in range(2)]
        for i, x in enumerate(arrs):
            idconv.fill_uniform(x, i, 1)
        ms = timed(idconv.hconv2d, arrs, 21, flush if fl else None)
        print(f"hconv2d 1023x512 {'flushed' if fl else 'no flush'}: {ms:.4f} ms per slab")
    # C5b's slab phase: 1535 such slabs; the default call for reference
    f = torch.empty((1023, 1023, 512), dtype=torch.complex128, device="cuda")
    g = torch.empty_like(f)
    idconv.fill_uniform(f, 0, 1)
    idconv.fill_uniform(g, 1, 1)
    ms = timed(idconv.hconv3d, (f, g), 3)
    print(f"hconv3d 1023^2 x 512: {ms:.3f} ms per call")


if __name__ == "__main__":
    main()
