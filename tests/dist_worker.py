"""Worker of the gloo tests of the distributed cconv3d / hconv3d decompositions.

Each rank follows the library's own host-side plan (idc_dist_plan, pure C
logic) for which x-planes it owns and which y-residues it receives (rows
[rank L, (rank+1) L) of every y stream, L = my / P), moves the
residue blocks with a real collective (torch.distributed all_to_all_single
over gloo), and evaluates the per-rank arithmetic with the oracle's implicit
equations (numpy; the GPU kernels are covered by the emulated-rank GPU test).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(rank, world, port, shape, outdir):
    import torch
    import torch.distributed as dist

    from oracle import implicit
    from paper_1008_1366_b200 import idconv
    import synthgen

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mx, my, mz = shape
    plan = idconv.dist_plan(mx, my, mz, world, rank)
    nx, nres, x0 = plan["nx"], plan["nres"], plan["x0"]
    f, g = synthgen.cconv3d_inputs(mx, my, mz)
    fl, gl = f[x0:x0 + nx], g[x0:x0 + nx]

    # phase A: fftpadBackward along y on the local planes (Eq. cconv1backward)
    def ypass(a):
        e, o = implicit.fftpad_backward(np.swapaxes(a, 1, 2))      # along y
        return np.concatenate([np.swapaxes(e, 1, 2), np.swapaxes(o, 1, 2)], axis=1)  # residues q = 0..2my-1

    L = my // world                                               # rows of each stream per rank

    def pack(streams, S=2):
        """rank p receives rows [p L, (p+1) L) of each of the S streams (q = s my + l)"""
        blocks = [np.concatenate([streams[:, s * my + p * L: s * my + (p + 1) * L, :] for s in range(S)], axis=1)
                  for p in range(world)]
        return torch.from_numpy(np.ascontiguousarray(np.stack(blocks)))   # [p][x][s L + l'][z]

    def unpack(back, S=2):
        return np.concatenate([np.concatenate([back[p][:, s * L:(s + 1) * L, :] for p in range(world)], axis=1)
                               for s in range(S)], axis=1)               # [x][s my + l][z]

    sf, sg = pack(ypass(fl)), pack(ypass(gl))
    rf, rg = torch.empty_like(sf), torch.empty_like(sg)
    dist.all_to_all_single(rf.view(torch.float64), sf.view(torch.float64))
    dist.all_to_all_single(rg.view(torch.float64), sg.view(torch.float64))
    # received [src][x_local][q'][z] == [x][q'][z]
    Rf = rf.numpy().reshape(mx, nres, mz)
    Rg = rg.numpy().reshape(mx, nres, mz)
    # phase B: 2D (x, z) convolution of every owned y-residue (Function cconv2)
    out = np.stack([implicit.cconv2d(Rf[:, q, :], Rg[:, q, :]) for q in range(nres)], axis=1)
    send_back = torch.from_numpy(np.ascontiguousarray(out.reshape(world, nx, nres, mz)))
    back = torch.empty_like(send_back)
    dist.all_to_all_single(back.view(torch.float64), send_back.view(torch.float64))
    # phase C: the streams from every source rank's block, fftpadForward along y
    streams = unpack(back.numpy())                                            # [x][2my][z]
    e, o = streams[:, :my, :], streams[:, my:, :]
    res = np.swapaxes(implicit.fftpad_forward(np.swapaxes(e, 1, 2), np.swapaxes(o, 1, 2)), 1, 2)
    np.save(os.path.join(outdir, f"rank{rank}.npy"), res)
    dist.barrier()
    dist.destroy_process_group()


def run_herm(rank, world, port, shape, outdir):
    """Hermitian decomposition (idc_hconv3d_dist): y-outer fft0pad streams,
    all-to-all, conv2 on the (x, z) plane of every owned y-residue, back."""
    import torch
    import torch.distributed as dist

    from oracle import implicit
    from paper_1008_1366_b200 import idconv
    import synthgen

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mx, my, mz = shape
    plan = idconv.dist_plan(mx, my, mz, world, rank, kind=idconv.HCONV3D)
    nx, nres, x0 = plan["nx"], plan["nres"], plan["x0"]
    f, g = synthgen.hconv3d_inputs(mx, my, mz)
    pad = lambda a: np.concatenate([a, np.zeros_like(a[:1])], axis=0)    # 2mx planes
    fl, gl = pad(f)[x0:x0 + nx], pad(g)[x0:x0 + nx]

    # phase A: fft0padBackward along the centered y axis (Eqs. fft0backwardA/B)
    def ypass(a):
        S = implicit.fft0pad_backward(np.moveaxis(a, 1, -1))          # r -> (nx, mz, my)
        return np.concatenate([np.moveaxis(S[r], -1, 1) for r in (-1, 0, 1)], axis=1)  # q = (r+1) my + l

    L = my // world

    def pack(streams, S=3):
        blocks = [np.concatenate([streams[:, s * my + p * L: s * my + (p + 1) * L, :] for s in range(S)], axis=1)
                  for p in range(world)]
        return torch.from_numpy(np.ascontiguousarray(np.stack(blocks)))

    def unpack(back, S=3):
        return np.concatenate([np.concatenate([back[p][:, s * L:(s + 1) * L, :] for p in range(world)], axis=1)
                               for s in range(S)], axis=1)

    sf, sg = pack(ypass(fl)), pack(ypass(gl))
    rf, rg = torch.empty_like(sf), torch.empty_like(sg)
    dist.all_to_all_single(rf.view(torch.float64), sf.view(torch.float64))
    dist.all_to_all_single(rg.view(torch.float64), sg.view(torch.float64))
    Rf = rf.numpy().reshape(2 * mx, nres, mz)
    Rg = rg.numpy().reshape(2 * mx, nres, mz)
    # phase B: conv2 (Function conv2) on the 2mx-1 valid x planes
    out = np.stack([pad(implicit.hconv2d(Rf[:-1, q, :], Rg[:-1, q, :])) for q in range(nres)], axis=1)
    send_back = torch.from_numpy(np.ascontiguousarray(out.reshape(world, nx, nres, mz)))
    back = torch.empty_like(send_back)
    dist.all_to_all_single(back.view(torch.float64), send_back.view(torch.float64))
    # phase C: fft0padForward along y
    streams = unpack(back.numpy())                                            # [x][3my][z]
    S = {r: np.moveaxis(streams[:, (r + 1) * my:(r + 2) * my, :], 1, -1) for r in (-1, 0, 1)}
    res = np.moveaxis(implicit.fft0pad_forward(S, my), -1, 1)
    np.save(os.path.join(outdir, f"rank{rank}.npy"), res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    rank, world, port = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    shape = tuple(int(x) for x in sys.argv[4].split(","))
    if len(sys.argv) > 6 and sys.argv[6] == "herm":
        run_herm(rank, world, port, shape, sys.argv[5])
    else:
        run(rank, world, port, shape, sys.argv[5])
