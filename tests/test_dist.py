"""Distributed 3D path.

* CPU, world_size 2 (gloo): the library's host-side decomposition plan drives
  a real 2-process all_to_all of the y-residue streams; the assembled result
  equals the oracle's direct sums.
* GPU: the exact CUDA phases of idc_cconv3d_dist run for P = 1, 2, 4, 8
  virtual ranks on one device (device copies stand in for the all-to-all),
  and the real NCCL path runs at P = 1.  (This box has one GPU; running
  ranks that wait on each other on one GPU is not allowed.)"""
import os
import subprocess
import sys

import numpy as np
import pytest

import synthgen
from oracle import direct, rel_l2

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("world,shape", [(2, (4, 4, 4)), (2, (8, 2, 4)), (4, (4, 4, 2))])
def test_decomposition_gloo(tmp_path, world, shape):
    port = 29500 + (os.getpid() % 400) + world
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "dist_worker.py"), str(r), str(world), str(port),
                               ",".join(map(str, shape)), str(tmp_path)]) for r in range(world)]
    for p in procs:
        assert p.wait(timeout=300) == 0
    res = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)], axis=0)
    f, g = synthgen.cconv3d_inputs(*shape)
    assert rel_l2(res, direct.cconv3d(f, g)) < 1e-13


@pytest.mark.parametrize("world,shape", [(2, (2, 2, 4)), (2, (4, 2, 2)), (4, (4, 4, 2))])
def test_hermitian_decomposition_gloo(tmp_path, world, shape):
    port = 29900 + (os.getpid() % 50) * 8 + world
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "dist_worker.py"), str(r), str(world), str(port),
                               ",".join(map(str, shape)), str(tmp_path), "herm"]) for r in range(world)]
    for p in procs:
        assert p.wait(timeout=300) == 0
    res = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)], axis=0)[:-1]  # drop padding plane
    f, g = synthgen.hconv3d_inputs(*shape)
    assert rel_l2(res, direct.hconv3d(f, g)) < 1e-13


def test_hermitian_plan_properties():
    from paper_1008_1366_b200 import idconv
    for (mx, my, mz, P) in [(512, 512, 512, 8), (4, 8, 4, 8), (2, 2, 2, 2)]:
        plans = [idconv.dist_plan(mx, my, mz, P, r, kind=idconv.HCONV3D) for r in range(P)]
        assert sum(p["nx"] for p in plans) == 2 * mx                 # 2mx-1 planes + 1 padding plane
        assert sum(p["nres"] for p in plans) == 3 * my               # every centered y-residue once
        assert all(p["S"] == p["nx"] * (2 * my - 1) * mz for p in plans)
    with pytest.raises(Exception):
        idconv.dist_plan(8, 2, 8, 4, 0, kind=idconv.HCONV3D)         # P must divide 3my
    assert idconv.workspace_bytes(idconv.HCONV3D, 4, 4, 4) > 0


def test_plan_properties():
    from paper_1008_1366_b200 import idconv
    for (mx, my, mz, P) in [(512, 512, 512, 8), (16, 8, 4, 4), (8, 8, 8, 1)]:
        plans = [idconv.dist_plan(mx, my, mz, P, r) for r in range(P)]
        assert sum(p["nx"] for p in plans) == mx
        assert sorted(p["x0"] for p in plans) == [r * mx // P for r in range(P)]
        assert sum(p["nres"] for p in plans) == 2 * my          # every y-residue owned exactly once
        assert all(p["blk"] == p["nx"] * p["nres"] * mz for p in plans)
    with pytest.raises(Exception):
        idconv.dist_plan(8, 8, 8, 3, 0)                          # P must be a power of two dividing mx


@pytest.mark.gpu
@pytest.mark.parametrize("P,shape", [(1, (8, 8, 8)), (2, (8, 4, 16)), (4, (16, 16, 8)), (8, (16, 8, 4)),
                                     (8, (64, 32, 32)), (8, (64, 64, 64))])
def test_emulated_ranks_gpu(P, shape):
    import torch
    from paper_1008_1366_b200 import idconv
    mx, my, mz = shape
    f, g = synthgen.cconv3d_inputs(*shape)
    nx = mx // P
    F = [torch.from_numpy(np.ascontiguousarray(f[r * nx:(r + 1) * nx])).cuda() for r in range(P)]
    G = [torch.from_numpy(np.ascontiguousarray(g[r * nx:(r + 1) * nx])).cuda() for r in range(P)]
    idconv.cconv3d_dist_emulated(F, G, mx, my, mz)
    res = np.concatenate([a.cpu().numpy() for a in F], axis=0)
    if mx * my * mz <= 4096:
        ref = direct.cconv3d(f, g)
        assert rel_l2(res, ref) < 1e-14
    else:
        idx = np.random.default_rng(3).choice(res.size, 64, replace=False)
        assert rel_l2(res.reshape(-1)[idx], direct.cconv_nd_at(f, g, idx)) < 1e-14
    # the single-GPU composition gives the same answer
    F1, G1 = torch.from_numpy(f.copy()).cuda(), torch.from_numpy(g.copy()).cuda()
    idconv.cconv3d(F1, G1)
    assert rel_l2(res, F1.cpu().numpy()) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", [False, True])
def test_nccl_single_rank_gpu(exchange):
    """One rank: the single-GPU composition (exchange=False, the default) and,
    through the test hook, the y-first phases with the NCCL all-to-alls."""
    import torch
    import torch.distributed as dist
    from paper_1008_1366_b200 import idconv
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = "29731" if exchange else "29735"
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = idconv.Comm()
        idconv.lib().idc_dist_force_exchange(int(exchange))
        shape = (16, 8, 16)
        f, g = synthgen.cconv3d_inputs(*shape)
        F, G = torch.from_numpy(f.copy()).cuda(), torch.from_numpy(g.copy()).cuda()
        idconv.cconv3d_dist(comm, F, G, *shape)
        torch.cuda.synchronize()
        assert rel_l2(F.cpu().numpy(), direct.cconv3d(f, g)) < 1e-14
        comm.close()
    finally:
        idconv.lib().idc_dist_force_exchange(0)
        dist.destroy_process_group()


def _herm_slabs(f, P):
    fp = np.concatenate([f, np.zeros_like(f[:1])], axis=0)           # 2mx planes (last = padding)
    nx = fp.shape[0] // P
    return [np.ascontiguousarray(fp[r * nx:(r + 1) * nx]) for r in range(P)]


@pytest.mark.gpu
@pytest.mark.parametrize("P,shape", [(1, (4, 4, 4)), (2, (4, 2, 8)), (4, (4, 4, 4)), (8, (4, 8, 4)),
                                     (8, (32, 16, 16)), (8, (64, 64, 64)), (4, (64, 64, 32))])
def test_hermitian_emulated_ranks_gpu(P, shape):
    import torch
    from paper_1008_1366_b200 import idconv
    mx, my, mz = shape
    f, g = synthgen.hconv3d_inputs(*shape)
    F = [torch.from_numpy(a).cuda() for a in _herm_slabs(f, P)]
    G = [torch.from_numpy(a).cuda() for a in _herm_slabs(g, P)]
    idconv.hconv3d_dist_emulated(F, G, mx, my, mz)
    res = np.concatenate([a.cpu().numpy() for a in F], axis=0)[:-1]
    if f.size <= 4096:
        assert rel_l2(res, direct.hconv3d(f, g)) < 1e-14
    else:
        idx = np.random.default_rng(5).choice(res.size, 64, replace=False)
        assert rel_l2(res.reshape(-1)[idx], direct.hconv3d_at(f, g, idx)) < 1e-14
    F1, G1 = torch.from_numpy(f.copy()).cuda(), torch.from_numpy(g.copy()).cuda()
    idconv.hconv3d(F1, G1)
    assert rel_l2(res, F1.cpu().numpy()) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", [False, True])
def test_hermitian_nccl_single_rank_gpu(exchange):
    import torch
    import torch.distributed as dist
    from paper_1008_1366_b200 import idconv
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = "29733" if exchange else "29737"
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = idconv.Comm()
        idconv.lib().idc_dist_force_exchange(int(exchange))
        shape = (8, 4, 16)
        f, g = synthgen.hconv3d_inputs(*shape)
        F, G = [torch.from_numpy(a).cuda() for a in _herm_slabs(f, 1)], [torch.from_numpy(a).cuda() for a in _herm_slabs(g, 1)]
        idconv.hconv3d_dist(comm, F[0], G[0], *shape)
        torch.cuda.synchronize()
        assert rel_l2(F[0].cpu().numpy()[:-1], direct.hconv3d(f, g)) < 1e-14
        comm.close()
    finally:
        idconv.lib().idc_dist_force_exchange(0)
        dist.destroy_process_group()


@pytest.mark.gpu
def test_exchange_spans_profiled_gpu():
    """The profiler files the NCCL exchanges of the forced P = 1 exchange path
    as "A2A" spans: 3 chunks there and 3 back for hconv3d (one per y stream),
    bytes = what this rank sends."""
    import torch
    import torch.distributed as dist
    from paper_1008_1366_b200 import idconv
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = "29741"
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = idconv.Comm()
        idconv.lib().idc_dist_force_exchange(1)
        shape = (8, 64, 16)
        f, g = synthgen.hconv3d_inputs(*shape)
        F, G = [torch.from_numpy(a).cuda() for a in _herm_slabs(f, 1)], [torch.from_numpy(a).cuda() for a in _herm_slabs(g, 1)]
        idconv.profile_begin()
        idconv.hconv3d_dist(comm, F[0], G[0], *shape)
        prof = idconv.profile_end()
        torch.cuda.synchronize()
        a2a = [r for r in prof if r["tag"] == "A2A"]
        assert len(a2a) == 1 and a2a[0]["n"] == 1 and a2a[0]["launches"] == 6, prof
        plan = idconv.dist_plan(*shape, 1, 0, kind=idconv.HCONV3D)
        words = plan["nx"] * plan["nres"] * shape[2]            # one rank's residues x its planes x mz
        assert a2a[0]["units"] == 16 * words * 3, (a2a, plan)   # both inputs there, one array back
        assert any(r["tag"] in ("K7", "K7s") for r in prof)
        assert rel_l2(F[0].cpu().numpy()[:-1], direct.hconv3d(f, g)) < 1e-14
        comm.close()
    finally:
        idconv.lib().idc_dist_force_exchange(0)
        dist.destroy_process_group()
