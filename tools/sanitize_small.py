"""Small calls of every kind for compute-sanitizer (one tool per run):
1D at m = 64 / 512 / 1024 / 4096, 2D/3D at sizes that reach the TMA pencils
and the m = 512 row kernels, the NEXT calls; results checked against the
oracle so a sanitizer-perturbed run still has to be right."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synthgen
from oracle import direct, rel_l2
from paper_1008_1366_b200 import idconv


def d(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


errs = {}
for m, B in [(64, 3), (512, 4), (1024, 2), (4096, 1)]:
    f, g, h = synthgen.hconv1d_inputs(m, B, roles=(0, 1, 2))
    F, G = d(f), d(g)
    idconv.cconv1d(F, G)
    errs[f"cconv1d {m}"] = rel_l2(F.cpu().numpy(), direct.cconv1d(f, g))
    F, G = d(f), d(g)
    idconv.hconv1d(F, G)
    errs[f"hconv1d {m}"] = rel_l2(F.cpu().numpy(), direct.hconv1d(f, g))
    F, G, H = d(f), d(g), d(h)
    idconv.tconv1d(F, G, H)
    errs[f"tconv1d {m}"] = rel_l2(F.cpu().numpy(), direct.tconv1d(f, g, h))
for mx, my in [(64, 64), (512, 8), (2048, 2)]:
    f, g = synthgen.cconv2d_inputs(mx, my, 1)
    F, G = d(f), d(g)
    idconv.cconv2d(F, G)
    errs[f"cconv2d {mx}x{my}"] = rel_l2(F.cpu().numpy()[0], direct.cconv2d(f[0], g[0]))
    f, g = synthgen.hconv2d_inputs(mx, my)
    F, G = d(f), d(g)
    idconv.hconv2d(F, G)
    errs[f"hconv2d {mx}x{my}"] = rel_l2(F.cpu().numpy(), direct.hconv2d(f, g))
for shape in [(8, 8, 512), (512, 4, 4), (64, 64, 8)]:
    f, g = synthgen.cconv3d_inputs(*shape)
    F, G = d(f), d(g)
    idconv.cconv3d(F, G)
    idx = np.random.default_rng(1).choice(f.size, 32, replace=False)
    errs[f"cconv3d {shape}"] = rel_l2(F.cpu().numpy().reshape(-1)[idx], direct.cconv_nd_at(f, g, idx))
    f, g = synthgen.hconv3d_inputs(*shape)
    F, G = d(f), d(g)
    idconv.hconv3d(F, G)
    idx = np.random.default_rng(2).choice(f.size, 32, replace=False)
    errs[f"hconv3d {shape}"] = rel_l2(F.cpu().numpy().reshape(-1)[idx], direct.hconv3d_at(f, g, idx))
w = synthgen.hconv2d_inputs(64, 64, roles=(0,))[0]
idconv.advection2d(d(w))
torch.cuda.synchronize()
bad = {k: v for k, v in errs.items() if not v < 1e-13}
print("max rel-L2", max(errs.values()), "bad:", bad)
sys.exit(1 if bad else 0)
