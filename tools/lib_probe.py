"""A/B of whole library builds through the raw C ABI (no binding, so builds
of other rounds with other exported symbols load too): bench.py's timing
(inputs restored and L2 flushed outside the events, events around the call)
for the small configs where host-side or event overhead could show.

usage: python tools/lib_probe.py LIB.so [LIB.so ...] [--profile] [--reps N]
"""
import ctypes
import sys

import torch

P, S, I = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int

CASES = [
    ("cconv1d 1024 x 32768", "idc_cconv1d", (32768, 1024), lambda L, p, w, nb: L.idc_cconv1d(p[0], p[1], 1024, 32768, w, nb, None), (0, 1024, 1, 1, 32768)),
    ("cconv2d 1024^2", "idc_cconv2d", (1, 1024, 1024), lambda L, p, w, nb: L.idc_cconv2d(p[0], p[1], 1024, 1024, 1, w, nb, None), (3, 1024, 1024, 1, 1)),
    ("cconv2d 64 x 256^2", "idc_cconv2d", (64, 256, 256), lambda L, p, w, nb: L.idc_cconv2d(p[0], p[1], 256, 256, 64, w, nb, None), (3, 256, 256, 1, 64)),
    ("hconv2d 4095 x 2048", "idc_hconv2d", (4095, 2048), lambda L, p, w, nb: L.idc_hconv2d(p[0], p[1], 2048, 2048, w, nb, None), (4, 2048, 2048, 1, 1)),
]


def setup(L):
    L.idc_cconv1d.argtypes = [P, P, S, S, P, S, P]
    L.idc_cconv2d.argtypes = [P, P, S, S, S, P, S, P]
    L.idc_hconv2d.argtypes = [P, P, S, S, P, S, P]
    L.idc_workspace_bytes.argtypes = [I, S, S, S, S]
    L.idc_workspace_bytes.restype = S
    for n in ("idc_cconv1d", "idc_cconv2d", "idc_hconv2d"):
        getattr(L, n).restype = I


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    profile = "--profile" in sys.argv
    reps = 30
    for a in sys.argv:
        if a.startswith("--reps="):
            reps = int(a.split("=")[1])
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for path in args:
        L = ctypes.CDLL(path)
        setup(L)
        use_prof = profile and hasattr(L, "idc_profile_begin")
        print(f"== {path}{' (profiler on)' if use_prof else ''}")
        for name, _, shape, fn, wargs in CASES:
            # kind ids of include/idconv.h
            kind = {"cconv1d": 0, "cconv2d": 3, "hconv2d": 4}[name.split()[0]]
            nb = L.idc_workspace_bytes(kind, *wargs[1:])
            w = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")
            f0 = torch.randn(shape, dtype=torch.complex128, device="cuda")
            g0 = torch.randn(shape, dtype=torch.complex128, device="cuda")
            f, g = f0.clone(), g0.clone()
            ptrs = [P(f.data_ptr()), P(g.data_ptr())]
            s = torch.cuda.current_stream()
            for _ in range(3):
                assert fn(L, ptrs, P(w.data_ptr()), nb) == 0
            if use_prof:
                L.idc_profile_begin()
            ts = []
            for _ in range(reps):
                f.copy_(f0)
                g.copy_(g0)
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                assert fn(L, ptrs, P(w.data_ptr()), nb) == 0
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            if use_prof:
                L.idc_profile_end.argtypes = [ctypes.c_char_p, S]
                L.idc_profile_end(None, 0)
            ts.sort()
            print(f"{name}: median {ts[len(ts) // 2]:.4f} ms, min {ts[0]:.4f} ms")
            del f, g, f0, g0, w
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
