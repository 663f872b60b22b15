"""BASELINE config 4 (3840x2160 stream, θps 12, θov 0.75, θsf 1, θit 64,
refinement 1/5) on the GPU — bit-exact, tolerance 0 (np.array_equal).

c4 is the only workload whose finest computed level (1920x1080, above 2^20
pixels) selects the two-blocks-per-SM 12-pixel lane kernel
(k_patch_gn<12, CODE, 2>) and the 1080-row SOR band split; these tests pin
both, end to end against the reference's own flow hash and against the
oracle, and stage by stage on a 1920x1080 level.
Reference: pipeline.py:150-163 (dis_flow), inverse_search.py:113-189,
variational.py:124-165, densification.py:110-191.
"""

import hashlib

import numpy as np
import pytest

from paper_1603_03590_b200.params import DisParams, VarParams
from tests.conftest import golden
from tools import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    return torch


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _np(t):
    return t.detach().cpu().numpy()


def test_c4_full_size_matches_reference_hash(torch):
    """Pair 0 of the c4 stream: sha256 of the CUDA flow == sha256 of the
    reference's flow on the same frames (tests/golden/full_hashes.npz)."""
    from paper_1603_03590_b200 import dis_flow_batch

    g = golden("full_hashes.npz")
    rows = [i for i, c in enumerate(g["cfg"]) if str(c) == "c4"]
    assert rows, "c4 hash missing from the golden"
    cfg = synth.CONFIGS["c4"]
    f1, f2 = synth.make_batch(cfg, seed=0, count=1, first=0)
    for i in rows:
        assert _sha(f1[0]) == str(g["f1_sha"][i]) and _sha(f2[0]) == str(g["f2_sha"][i])
    flow = dis_flow_batch(f1, f2, synth.dis_params(cfg)).cpu().numpy()
    for i in rows:
        assert _sha(flow[int(g["pair"][i])]) == str(g["flow_sha"][i])


def test_c4_batched_pairs_vs_oracle(torch, orc):
    """Two consecutive c4 pairs (frames 0-1, 1-2 of a seed-3 stream) in one
    batch against the oracle: batching does not couple the pairs."""
    from paper_1603_03590_b200 import dis_flow_batch

    cfg = synth.CONFIGS["c4"]
    f1, f2 = synth.make_batch(cfg, seed=3, count=2)
    params = synth.dis_params(cfg)
    flow = dis_flow_batch(f1, f2, params).cpu().numpy()
    want = orc.dis_flow_batch_f32(f1, f2, params)
    for k in range(2):
        assert np.array_equal(flow[k], want[k]), k


@pytest.fixture(scope="module")
def level_1080(torch):
    """A 1920x1080 level pair (c4's level 1): frames of a c3-like pair with
    up to 32 px motion, and a coarse flow for the search's init."""
    cfg = synth.CONFIGS["c4"]
    f1, f2, gt = synth.make_pair(11, 1080, 1920, 32.0, True, 32.0)
    coarse = np.ascontiguousarray(gt[::2, ::2] * 0.5)  # a 960x540 stand-in
    return cfg, f1, f2, coarse


def test_c4_level_patch_search_and_densify_vs_oracle(torch, orc, level_1080):
    """θps 12 / θov 0.75 / θit 64 on a 2.07 Mpixel level (the lane kernel's
    two-blocks-per-SM instance), every patch output and the densified field
    bit-exact against the oracle."""
    from paper_1603_03590_b200 import stages

    cfg, f1, f2, coarse = level_1080
    params = DisParams(patch_size=12, overlap=0.75, iterations=64, finest_scale=0,
                       coarsest_scale=1)
    l1 = stages.build_pyramid(f1[None], 0)[0]
    l2 = stages.build_pyramid(f2[None], 0)[0]
    c = torch.tensor(coarse, device="cuda")
    cu, cv = c[..., 0][None].contiguous(), c[..., 1][None].contiguous()
    r = stages.patch_search(l1, l2["img"], params, cu, cv)
    assert len(r["x_origins"]) * len(r["y_origins"]) > 200_000
    ref = orc.build_pyramid(f1, 0)[0]
    qry = orc.build_pyramid(f2, 0)[0]
    xo, sp = orc.axis_origins(1920, 12, 0.75)
    yo, _ = orc.axis_origins(1080, 12, 0.75)
    assert np.array_equal(r["x_origins"], xo) and np.array_equal(r["y_origins"], yo)
    init = orc.init_patches(xo, yo, 12, coarse)
    assert np.array_equal(np.stack([_np(r["init_u"])[0], _np(r["init_v"])[0]], -1), init)
    want = orc.patch_search(ref[0], ref[1], ref[2], qry[0], xo, yo, 12, init, 64)
    assert np.array_equal(_np(r["valid"])[0].astype(bool), want["valid"])
    disp = np.stack([_np(r["u"])[0], _np(r["v"])[0]], -1)
    assert np.array_equal(disp, want["disp"])
    assert np.array_equal(_np(r["off"])[0], want["offset"])
    fu, fv = stages.densify(l1["img"], l2["img"], params, r["u"], r["v"], r["off"])
    dense = orc.densify(ref[0], qry[0], xo, yo, 12, want["disp"], want["offset"])
    assert np.array_equal(np.stack([_np(fu)[0], _np(fv)[0]], -1), dense)


def test_c4_level_refine_vs_oracle(torch, orc, level_1080):
    """Refinement of a 1080-row level (the nine-band cluster split of the
    wavefront SOR), 1 outer / 5 inner and 2 outer / 5 inner."""
    from paper_1603_03590_b200 import stages

    cfg, f1, f2, coarse = level_1080
    init = np.repeat(np.repeat(coarse, 2, axis=0), 2, axis=1) * 2.0
    l1 = stages.build_pyramid(f1[None], 0)[0]
    l2 = stages.build_pyramid(f2[None], 0)[0]
    ref = orc.build_pyramid(f1, 0)[0]
    qry = orc.build_pyramid(f2, 0)[0]
    t = torch.tensor(init, device="cuda")
    u0, v0 = t[..., 0][None].contiguous(), t[..., 1][None].contiguous()
    vp = VarParams()
    for outer in (1, 2):
        u, v = stages.refine(u0, v0, l1, l2, DisParams(variational=vp), outer)
        want = orc.refine(init, ref, qry, vp, outer)
        assert np.array_equal(np.stack([_np(u)[0], _np(v)[0]], -1), want), outer
