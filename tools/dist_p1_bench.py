"""Time the distributed 3D calls on a one-rank communicator with the exchange
phases forced (idc_dist_force_exchange): y pass into the send blocks, NCCL
self all-to-all, (x, z) convolutions, all-to-all back, y pass from the
returned blocks -- against the single-GPU call on the same arrays."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from paper_1008_1366_b200 import idconv

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29771")
dist.init_process_group("gloo", rank=0, world_size=1)
comm = idconv.Comm()
for kind, m in (("cconv3d", 512), ("hconv3d", 512)):
    herm = kind == "hconv3d"
    shape = (2 * m, 2 * m - 1, m) if herm else (m, m, m)
    src = [torch.empty(shape, dtype=torch.complex128, device="cuda") for _ in range(2)]
    for i, a in enumerate(src):
        idconv.fill_uniform(a, i, 1)
        a /= 1e3
    work = [torch.empty_like(a) for a in src]
    fn = idconv.hconv3d_dist if herm else idconv.cconv3d_dist
    single = idconv.hconv3d if herm else idconv.cconv3d
    for force in (1, 0):
        idconv.lib().idc_dist_force_exchange(force)
        ts = []
        for r in range(4):
            for s_, d_ in zip(src, work):
                d_.copy_(s_)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(comm, work[0], work[1], m, m, m)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"{kind}_dist P=1 force_exchange={force}: {min(ts[1:]):.2f} ms", flush=True)
    a = [s_[:-1].contiguous() if herm else s_.clone() for s_ in src]
    ts = []
    for r in range(4):
        b = [x.clone() for x in a]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        single(*b)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{kind} single GPU: {min(ts[1:]):.2f} ms", flush=True)
    del src, work, a
    torch.cuda.empty_cache()
idconv.lib().idc_dist_force_exchange(0)
comm.close()
dist.destroy_process_group()
