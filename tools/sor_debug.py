"""Debug: GPU refine vs oracle refine on small levels; prints the first
mismatching pixels (row, col) per case.  python tools/sor_debug.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import oracle as orc
from paper_1603_03590_b200 import stages
from paper_1603_03590_b200.params import DisParams, VarParams

for (H, W, sweeps) in [(5, 6, 1), (13, 32, 1), (13, 32, 2), (13, 32, 5), (40, 20, 1), (70, 30, 3)]:
    rng = np.random.default_rng(5)
    f1 = rng.uniform(0, 255, (1, H, W))
    f2 = np.roll(f1, 1, axis=2) + rng.normal(0, 2, (1, H, W))
    init = rng.normal(0, 1.5, (1, H, W, 2))
    l1 = stages.build_pyramid(f1, 0)[0]
    l2 = stages.build_pyramid(f2, 0)[0]
    t = torch.tensor(init, device="cuda")
    u0, v0 = t[..., 0].contiguous(), t[..., 1].contiguous()
    vp = VarParams(inner_sor_iters=sweeps)
    u, v = stages.refine(u0, v0, l1, l2, DisParams(variational=vp), 1)
    got = np.stack([u.cpu().numpy(), v.cpu().numpy()], -1)[0]
    want = orc.refine(init[0], orc.build_pyramid(f1[0], 0)[0], orc.build_pyramid(f2[0], 0)[0], vp, 1)
    bad = np.argwhere(np.any(got != want, axis=-1))
    print(f"H={H} W={W} S={sweeps}: {len(bad)} bad of {H*W}; first {bad[:6].tolist()}", flush=True)
    if len(bad):
        r, c = bad[0]
        print("   got", got[r, c], "want", want[r, c], "init", init[0, r, c])
