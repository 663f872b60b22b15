"""SOR band splits and sweep groups against the oracle (GPU).

The wavefront SOR splits a level's rows over a cluster of CTAs (halo rows
exchanged through distributed shared memory) and gives each thread a group
of sweeps.  The
split and the group size are picked from the batch and level sizes, so the
parity tests at their natural sizes see only a few combinations; here the
experiment knobs DIS_SOR_CLUSTER / DIS_SOR_P (read once per process) force
1..7 bands and 1/2/S sweeps per thread in subprocesses, each compared
bit for bit with the oracle's refine (variational.py:220-275)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
from paper_1603_03590_b200 import stages
from paper_1603_03590_b200.params import DisParams, VarParams
rng = np.random.default_rng(5)
H, W, B = 200, 72, 2
f1 = rng.uniform(0, 255, (B, H, W))
f2 = np.roll(f1, 1, axis=2) + rng.normal(0, 2, (B, H, W))
init = rng.normal(0, 1.5, (B, H, W, 2))
l1 = stages.build_pyramid(f1, 0)[0]
l2 = stages.build_pyramid(f2, 0)[0]
t = torch.tensor(init, device="cuda")
u0, v0 = t[..., 0].contiguous(), t[..., 1].contiguous()
vp = VarParams(inner_sor_iters=int(sys.argv[2]))
u, v = stages.refine(u0, v0, l1, l2, DisParams(variational=vp), 1)
np.save(sys.argv[3], np.stack([u.cpu().numpy(), v.cpu().numpy()], -1))
"""


@pytest.fixture(scope="module")
def reference():
    from oracle import oracle as orc

    rng = np.random.default_rng(5)
    H, W, B = 200, 72, 2
    f1 = rng.uniform(0, 255, (B, H, W))
    f2 = np.roll(f1, 1, axis=2) + rng.normal(0, 2, (B, H, W))
    init = rng.normal(0, 1.5, (B, H, W, 2))
    from paper_1603_03590_b200.params import VarParams

    out = {}
    for sweeps in (5, 3):
        vp = VarParams(inner_sor_iters=sweeps)
        out[sweeps] = np.stack([
            orc.refine(init[b], orc.build_pyramid(f1[b], 0)[0], orc.build_pyramid(f2[b], 0)[0],
                       vp, 1) for b in range(B)])
    return out


@pytest.mark.parametrize("bands,group,sweeps", [(2, 0, 5), (3, 1, 5), (4, 2, 5),
                                                (7, 0, 5), (5, 5, 5), (3, 2, 3), (6, 1, 3)])
def test_band_split_and_sweep_groups_match_oracle(reference, tmp_path, bands, group, sweeps):
    env = dict(os.environ)
    env["DIS_SOR_CLUSTER"] = str(bands)
    if group:
        env["DIS_SOR_P"] = str(group)
    else:
        env.pop("DIS_SOR_P", None)
    out = tmp_path / "flow.npy"
    subprocess.run([sys.executable, "-c", CHILD, ROOT, str(sweeps), str(out)], env=env,
                   check=True, timeout=300, cwd=ROOT)
    assert np.array_equal(np.load(out), reference[sweeps])


# The ring is filled by one TMA box per diagonal: the box holds the band's
# rows rounded up to 4 (at most 128), the row below the band is a second
# 16-byte box, rows past the level are zero-filled by the TMA unit and slots
# of pixels outside the level are masked in the kernel.  Shapes at those
# edges: 124- and 128-row bands (the largest box), 125 rows, band heights
# whose ring rows need rounding, levels much wider / much taller than the
# other dimension (most of a diagonal's slots outside the level), and the
# tallest supported levels (16 bands of 128 rows: 2048 rows; 2033).
CHILD_SHAPE = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1])
from paper_1603_03590_b200 import stages
from paper_1603_03590_b200.params import DisParams, VarParams
H, W, B = int(sys.argv[2]), int(sys.argv[3]), 2
rng = np.random.default_rng(H * 1000 + W)
f1 = rng.uniform(0, 255, (B, H, W))
f2 = np.roll(f1, 1, axis=2) + rng.normal(0, 2, (B, H, W))
init = rng.normal(0, 1.5, (B, H, W, 2))
l1 = stages.build_pyramid(f1, 0)[0]
l2 = stages.build_pyramid(f2, 0)[0]
t = torch.tensor(init, device="cuda")
u, v = stages.refine(t[..., 0].contiguous(), t[..., 1].contiguous(), l1, l2, DisParams(), 1)
np.save(sys.argv[4], np.stack([u.cpu().numpy(), v.cpu().numpy()], -1))
"""


@pytest.mark.parametrize("H,W,bands", [(124, 40, 1), (125, 40, 0), (123, 37, 1), (94, 61, 2),
                                       (128, 40, 1), (17, 300, 0), (250, 9, 0), (2048, 24, 0),
                                       (2033, 20, 0)])
def test_tma_ring_edges_match_oracle(tmp_path, H, W, bands):
    from oracle import oracle as orc
    from paper_1603_03590_b200.params import VarParams

    env = dict(os.environ)
    env.pop("DIS_SOR_P", None)
    if bands:
        env["DIS_SOR_CLUSTER"] = str(bands)
    else:
        env.pop("DIS_SOR_CLUSTER", None)
    out = tmp_path / "flow.npy"
    subprocess.run([sys.executable, "-c", CHILD_SHAPE, ROOT, str(H), str(W), str(out)], env=env,
                   check=True, timeout=300, cwd=ROOT)
    B = 2
    rng = np.random.default_rng(H * 1000 + W)
    f1 = rng.uniform(0, 255, (B, H, W))
    f2 = np.roll(f1, 1, axis=2) + rng.normal(0, 2, (B, H, W))
    init = rng.normal(0, 1.5, (B, H, W, 2))
    want = np.stack([orc.refine(init[b], orc.build_pyramid(f1[b], 0)[0],
                                orc.build_pyramid(f2[b], 0)[0], VarParams(), 1)
                     for b in range(B)])
    assert np.array_equal(np.load(out), want)
