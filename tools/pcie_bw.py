"""Host<->device copy ceiling of this box (context for bench.py's e2e leg):
pinned host buffers, one large cudaMemcpyAsync per direction, and both
directions at once on two streams.  Prints one JSON line (GB/s)."""
import json

import torch


def _bw(fn, nbytes, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        best = t if best is None else min(best, t)
    return nbytes / best / 1e9


def main():
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h2d = _bw(lambda: d.copy_(h, non_blocking=True), n)
    d2h = _bw(lambda: h.copy_(d, non_blocking=True), n)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    duplex = _bw(both, 2 * n)
    print(json.dumps({"h2d_gbs": round(h2d, 2), "d2h_gbs": round(d2h, 2), "duplex_total_gbs": round(duplex, 2),
                      "bytes": n}))


if __name__ == "__main__":
    main()
