"""§8(f) "next" rows on the GPU through the C ABI, against the reference's
goldens and the oracle — bit-exact (tolerance 0: np.array_equal)."""

import numpy as np
import pytest

from tests.conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    return torch


# ---- compose_flows (pipeline.py:186-199) ----------------------------------

def test_compose_flows_goldens(torch):
    from paper_1603_03590_b200 import compose_flows

    g = golden("next_compose.npz")
    for k in range(3):
        got = compose_flows(g[f"ab{k}"], g[f"bc{k}"])
        assert isinstance(got, np.ndarray) and got.dtype == np.float64
        assert np.array_equal(got, g[f"out{k}"]), k


def test_compose_flows_batched_torch_vs_oracle(torch, orc):
    from paper_1603_03590_b200 import compose_flows

    rng = np.random.default_rng(5)
    ab = rng.normal(0, 6, (3, 64, 96, 2))
    bc = rng.normal(0, 6, (3, 64, 96, 2))
    got = compose_flows(torch.from_numpy(ab).cuda(), torch.from_numpy(bc).cuda())
    assert got.is_cuda
    got = got.cpu().numpy()
    for i in range(3):
        assert np.array_equal(got[i], orc.compose_flows(ab[i], bc[i])), i


def test_compose_flows_errors(torch):
    from paper_1603_03590_b200 import compose_flows

    with pytest.raises(ValueError):
        compose_flows(np.zeros((4, 5, 2)), np.zeros((4, 6, 2)))


def _params(g):
    from tests.test_next_oracle import params_from

    return params_from(g)


# ---- stereo (pipeline.py:166-183) ------------------------------------------

@pytest.mark.parametrize("k", range(4))
def test_stereo_end_to_end_goldens(torch, k):
    from paper_1603_03590_b200 import dis_stereo

    g = golden(f"next_stereo_{k}.npz")
    flow = dis_stereo(g["f1"], g["f2"], _params(g))
    assert np.array_equal(flow, g["flow"])
    assert not np.any(flow[..., 1])


def test_stereo_batch_vs_oracle_and_host_path(torch, orc):
    from paper_1603_03590_b200 import FlowEngine, DisParams, dis_stereo_batch
    from tools import synth

    p = DisParams.preset(3, stereo=True, coarsest_scale=4)
    pairs = [synth.make_stereo_pair(30 + i, 218, 512, 16.0) for i in range(3)]
    f1 = np.stack([a for a, _, _ in pairs])
    f2 = np.stack([b for _, b, _ in pairs])
    got = dis_stereo_batch(f1, f2, p).cpu().numpy()
    for i in range(3):
        assert np.array_equal(got[i], orc.dis_stereo(f1[i], f2[i], p)), i
    eng = FlowEngine(3, 218, 512, p, stereo=True)
    assert np.array_equal(eng.run_host(f1, f2), got)


def test_stereo_graph_replays_and_pinned_host_dtypes(torch):
    # the graph-replayed device path and the captured host path, stereo
    # engines and every frame dtype, against the eager device result
    from paper_1603_03590_b200 import FlowEngine, DisParams
    from tools import synth

    p = DisParams.preset(3, stereo=True, coarsest_scale=3)
    pairs = [synth.make_stereo_pair(40 + i, 109, 256, 8.0) for i in range(2)]
    f1 = np.stack([a for a, _, _ in pairs])
    f2 = np.stack([b for _, b, _ in pairs])
    eng = FlowEngine(2, 109, 256, p, stereo=True)
    for dt in (np.float32, np.float64, np.uint8):
        a = np.clip(f1, 0, 255).astype(dt)
        b = np.clip(f2, 0, 255).astype(dt)
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        want = eng.run(ta, tb).cpu().numpy()
        out = torch.empty((2, 109, 256, 2), dtype=torch.float64, device="cuda")
        s = torch.cuda.Stream()
        for _ in range(2):
            eng.run(ta, tb, out=out, stream=s, graph=True)
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy(), want), dt
        pa = torch.from_numpy(a).pin_memory()
        pb = torch.from_numpy(b).pin_memory()
        po = torch.empty((2, 109, 256, 2), dtype=torch.float64).pin_memory()
        for _ in range(3):  # eager, capture, replay
            po.zero_()
            eng.run_host(pa.numpy(), pb.numpy(), out=po.numpy())
            assert np.array_equal(po.numpy(), want), dt


def test_stereo_mode_params_rejected_by_dis_flow(torch):
    from paper_1603_03590_b200 import DisParams, dis_flow

    a = np.zeros((64, 64), dtype=np.float32)
    with pytest.raises(ValueError):
        dis_flow(a, a, DisParams.preset(2, stereo=True, coarsest_scale=2))


def test_stereo_stages(torch):
    """horizontal-only refine (variational.py:161) through dis_refine."""
    from paper_1603_03590_b200 import DisParams, VarParams, stages

    g = golden("next_stereo_stages.npz")
    r = golden("refine.npz")
    lv1 = stages.build_pyramid(r["f1"], 0)[0]
    lv2 = stages.build_pyramid(r["f2"], 0)[0]
    init = r["init"]
    fu = torch.from_numpy(np.ascontiguousarray(init[None, ..., 0])).cuda()
    fv = torch.from_numpy(np.ascontiguousarray(init[None, ..., 1])).cuda()
    p = DisParams(mode="stereo", variational=VarParams())
    u, v = stages.refine(fu, fv, lv1, lv2, p, 2)
    got = np.stack([u[0].cpu().numpy(), v[0].cpu().numpy()], axis=-1)
    assert np.array_equal(got, g["refined_h"])


# ---- bidirectional densification (densification.py:131-153, 194-234) ------

def test_densify_bidirectional_stage_goldens(torch, orc):
    from paper_1603_03590_b200 import DisParams, stages

    g = golden("next_bidir_stage.npz")
    lv1 = stages.build_pyramid(g["f1"], 0)[0]
    lv2 = stages.build_pyramid(g["f2"], 0)[0]
    for k in range(3):
        p = DisParams(patch_size=int(g[f"ps{k}"]), overlap=float(g[f"ov{k}"]))
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)[None]).cuda()  # noqa: E731
        fd, bd = g[f"fdisp{k}"], g[f"bdisp{k}"]
        u, v = stages.densify_bidirectional(lv1["img"], lv2["img"], p, t(fd[:, 0]), t(fd[:, 1]),
                                            t(g[f"foff{k}"]), t(bd[:, 0]), t(bd[:, 1]),
                                            t(g[f"boff{k}"]))
        got = np.stack([u[0].cpu().numpy(), v[0].cpu().numpy()], axis=-1)
        assert np.array_equal(got, g[f"flow{k}"]), k


def test_densify_bidirectional_overflow_tile(torch, orc):
    """Every backward patch displaced onto the same tile: the tile's list
    exceeds the shared-memory capacity and the kernel falls back to the
    in-order scan of all patches — still the reference's sums."""
    from paper_1603_03590_b200 import DisParams, stages

    rng = np.random.default_rng(11)
    h, w, ps = 200, 240, 4
    img1 = rng.uniform(0, 255, (h, w))
    img2 = rng.uniform(0, 255, (h, w))
    p = DisParams(patch_size=ps, overlap=0.75)
    xo = stages.grid_axis(w, ps, 0.75)
    yo = stages.grid_axis(h, ps, 0.75)
    gx, gy = np.meshgrid(xo.astype(np.float64), yo.astype(np.float64))
    n = gx.size
    assert n > 2048
    fd = rng.normal(0, 1, (n, 2))
    bd = np.stack([100.3 - gx.ravel(), 50.6 - gy.ravel()], -1)  # all land at (100.3, 50.6)
    fo, bo = rng.normal(0, 1, n), rng.normal(0, 1, n)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)[None]).cuda()  # noqa: E731
    u, v = stages.densify_bidirectional(t(img1), t(img2), p, t(fd[:, 0]), t(fd[:, 1]), t(fo),
                                        t(bd[:, 0]), t(bd[:, 1]), t(bo))
    got = np.stack([u[0].cpu().numpy(), v[0].cpu().numpy()], axis=-1)
    want = orc.densify_bidirectional(img1, img2, xo, yo, fd, fo, xo, yo, bd, bo, ps)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("k", range(4))
def test_bidirectional_end_to_end_goldens(torch, k):
    from paper_1603_03590_b200 import dis_flow

    g = golden(f"next_bidir_{k}.npz")
    assert np.array_equal(dis_flow(g["f1"], g["f2"], _params(g)), g["flow"])


def test_bidirectional_batch_full_size_vs_oracle(torch, orc):
    import dataclasses

    from paper_1603_03590_b200 import dis_flow_batch
    from tools import synth

    cfg = synth.CONFIGS["c1"]
    f1, f2 = synth.make_batch(cfg, seed=40, count=2)
    p = dataclasses.replace(synth.dis_params(cfg), bidirectional=True)
    got = dis_flow_batch(f1, f2, p).cpu().numpy()
    for i in range(2):
        assert np.array_equal(got[i], orc.dis_flow(f1[i], f2[i], p)), i


# ---- sparse correspondences (pipeline.py:202-287) ---------------------------

@pytest.mark.parametrize("name", ["dense", "chain", "chain_s0", "dense_bidir"])
def test_sparse_correspondences_goldens(torch, name):
    from paper_1603_03590_b200 import sparse_correspondences
    from tests.test_next_oracle import sparse_params

    g = golden("next_sparse.npz")
    m = sparse_correspondences(g["f1"], g["f2"], g["seeds"], sparse_params(g, name))
    assert np.array_equal(np.array([x.valid for x in m]), g[f"{name}_valid"])
    assert np.array_equal(np.array([x.displacement for x in m]), g[f"{name}_disp"])
    assert np.array_equal(np.array([x.seed for x in m]), g[f"{name}_seed"])


def test_sparse_no_valid_seed_and_single_seed(torch):
    from paper_1603_03590_b200 import DisParams, sparse_correspondences

    a = np.random.default_rng(3).uniform(0, 255, (64, 96)).astype(np.float32)
    p = DisParams(coarsest_scale=2, finest_scale=1, use_densification=False)
    m = sparse_correspondences(a, a, [(-1.0, 3.0), (96.0, 3.0)], p)
    assert [x.valid for x in m] == [False, False]
    assert all(x.displacement == (0.0, 0.0) for x in m)
    m = sparse_correspondences(a, a, (10.0, 20.0), p)  # a single seed (atleast_2d)
    assert len(m) == 1 and m[0].valid


# ---- pyramid-level entry point (pipeline.py:136-147, core.py:33-128) --------

def test_build_pyramid_matches_reference_golden(torch):
    from paper_1603_03590_b200 import build_pyramid

    g = golden("pyramid.npz")
    pyr = build_pyramid(g["img"], 4)
    assert len(pyr) == 5 and pyr.downscale == 2
    for s in range(5):
        lv = pyr[s]
        assert lv.scale_index == s and lv.width == g[f"L{s}_img"].shape[1]
        assert np.array_equal(lv.image.cpu().numpy(), g[f"L{s}_img"]), s
        assert np.array_equal(lv.grad_x.cpu().numpy(), g[f"L{s}_gx"]), s
        assert np.array_equal(lv.grad_y.cpu().numpy(), g[f"L{s}_gy"]), s


@pytest.mark.parametrize("case", ["c1", "c2"])
def test_dis_flow_on_pyramids_equals_dis_flow(torch, orc, case):
    """Our GPU pyramids and numpy pyramids in the reference's layout (oracle)
    both give the reference's flow."""
    from paper_1603_03590_b200 import (ImagePyramid, PyramidLevel, build_pyramid,
                                       dis_flow_on_pyramids)
    from tests.test_gpu_parity import _params_from

    g = golden(f"e2e_{case}.npz")
    p = _params_from(g)
    got = dis_flow_on_pyramids(build_pyramid(g["f1"], p.coarsest_scale),
                               build_pyramid(g["f2"], p.coarsest_scale), p)
    assert got.is_cuda
    assert np.array_equal(got.cpu().numpy(), g["flow"])

    def np_pyr(f):
        lv = orc.build_pyramid(f, p.coarsest_scale)
        return ImagePyramid(tuple(PyramidLevel(i, gx, gy, s) for s, (i, gx, gy) in
                                  enumerate(lv)), 2)

    got = dis_flow_on_pyramids(np_pyr(g["f1"]), np_pyr(g["f2"]), p)
    assert isinstance(got, np.ndarray) and np.array_equal(got, g["flow"])


def test_dis_flow_on_pyramids_errors_and_warmup(torch):
    from paper_1603_03590_b200 import (DisParams, ParameterError, build_pyramid,
                                       dis_flow_on_pyramids, warmup)

    warmup()
    a = build_pyramid(np.random.default_rng(0).uniform(0, 255, (40, 64)), 2)
    b = build_pyramid(np.random.default_rng(1).uniform(0, 255, (40, 66)), 2)
    with pytest.raises(ValueError):
        dis_flow_on_pyramids(a, b, DisParams(coarsest_scale=2, finest_scale=1))
    with pytest.raises(ValueError):
        dis_flow_on_pyramids(a, a, DisParams.preset(2, stereo=True, coarsest_scale=2))
    with pytest.raises(ValueError):  # coarsest level 16x10 cannot hold a 12 px patch
        dis_flow_on_pyramids(a, a, DisParams(patch_size=12, coarsest_scale=2, finest_scale=1))
    with pytest.raises(ParameterError):
        build_pyramid(np.zeros((8, 8)), -1)
