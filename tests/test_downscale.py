"""downscale > 2 — the pyramid factor of DisParams (core.py:88-128, 250,
305-306): box means over k x k blocks, init_patches at centre / k scaled by k
(densification.py:82-95), upsample_flow by k (core.py:178-190) and the sparse
chain's k^s scaling (pipeline.py:202-231).  Goldens from the reference itself
(oracle/gen_golden.py gen_downscale -> tests/golden/downscale.npz); the C
oracle is pinned to them on the CPU, the CUDA path bit-exact on the GPU."""

import numpy as np
import pytest

from paper_1603_03590_b200.params import DisParams, VarParams
from tests.conftest import golden

FLOW_CASES = ["f3", "f3_default_outer", "f4", "f3_s0", "f3_bidir"]


def params_of(g, name):
    outer = int(g[f"{name}_outer"])
    vp = (VarParams(outer_iters_fixed=None if outer < 0 else outer)
          if int(g[f"{name}_variational"]) else None)
    return DisParams(patch_size=int(g[f"{name}_patch_size"]),
                     overlap=float(g[f"{name}_overlap"]),
                     iterations=int(g[f"{name}_iterations"]),
                     finest_scale=int(g[f"{name}_finest"]),
                     coarsest_scale=int(g[f"{name}_coarsest"]),
                     downscale=int(g[f"{name}_downscale"]),
                     use_mean_normalization=bool(int(g[f"{name}_mean_norm"])),
                     residual_norm=str(g[f"{name}_norm"]), variational=vp,
                     mode=str(g[f"{name}_mode"]),
                     bidirectional=bool(int(g[f"{name}_bidirectional"])))


def stereo_params():
    return DisParams(patch_size=8, overlap=0.5, iterations=16, finest_scale=1, coarsest_scale=2,
                     downscale=3, mode="stereo", variational=VarParams(outer_iters_fixed=1))


def sparse_params(dens):
    return DisParams(patch_size=8, overlap=0.5, iterations=32, finest_scale=1, coarsest_scale=2,
                     downscale=3, use_densification=dens,
                     variational=VarParams(outer_iters_fixed=1))


# ---- the oracle pinned to the reference (CPU) -------------------------------

@pytest.mark.parametrize("k", [3, 4, 8, 9])
def test_box_pyramid_oracle(orc, k):
    g = golden("downscale.npz")
    n = 3 if k < 8 else 2
    lv = orc.build_pyramid(g[f"pyr{k}_img"], n - 1, downscale=k)
    for s in range(n):
        assert np.array_equal(lv[s][0], g[f"pyr{k}_L{s}"]), (k, s)
        assert np.array_equal(lv[s][1], g[f"pyr{k}_L{s}_gx"]), (k, s)
        assert np.array_equal(lv[s][2], g[f"pyr{k}_L{s}_gy"]), (k, s)


@pytest.mark.parametrize("name", FLOW_CASES)
def test_flow_oracle(orc, name):
    g = golden("downscale.npz")
    out = orc.dis_flow(g[f"{name}_f1"], g[f"{name}_f2"], params_of(g, name))
    assert np.array_equal(out, g[f"{name}_flow"])


def test_stereo_and_sparse_oracle(orc):
    g = golden("downscale.npz")
    assert np.array_equal(orc.dis_stereo(g["st3_f1"], g["st3_f2"], stereo_params()),
                          g["st3_flow"])
    for name, dens in (("sp_dense", True), ("sp_chain", False)):
        disp, valid = orc.sparse_correspondences(g["sp_f1"], g["sp_f2"], g["sp_seeds"],
                                                 sparse_params(dens))
        assert np.array_equal(disp, g[f"{name}_disp"]), name
        assert np.array_equal(valid, g[f"{name}_valid"]), name


# ---- the CUDA path (GPU) ----------------------------------------------------

@pytest.fixture(scope="module")
def torch():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    return torch


@pytest.mark.gpu
@pytest.mark.parametrize("k", [3, 4, 8, 9])
def test_box_pyramid_gpu(torch, k):
    from paper_1603_03590_b200 import stages

    g = golden("downscale.npz")
    n = 3 if k < 8 else 2
    img = g[f"pyr{k}_img"][None]
    for second in (True, False):
        lv = stages.build_pyramid(img, n - 1, second_derivatives=second, downscale=k)
        for s in range(n):
            assert np.array_equal(lv[s]["img"].cpu().numpy()[0], g[f"pyr{k}_L{s}"]), (k, s)
            assert np.array_equal(lv[s]["gx"].cpu().numpy()[0], g[f"pyr{k}_L{s}_gx"]), (k, s)
            assert np.array_equal(lv[s]["gy"].cpu().numpy()[0], g[f"pyr{k}_L{s}_gy"]), (k, s)


@pytest.mark.gpu
@pytest.mark.parametrize("name", FLOW_CASES)
def test_flow_gpu(torch, name):
    from paper_1603_03590_b200 import dis_flow, dis_flow_batch

    g = golden("downscale.npz")
    p = params_of(g, name)
    assert np.array_equal(dis_flow(g[f"{name}_f1"], g[f"{name}_f2"], p), g[f"{name}_flow"])
    two = dis_flow_batch(np.stack([g[f"{name}_f1"]] * 2), np.stack([g[f"{name}_f2"]] * 2), p)
    assert np.array_equal(two.cpu().numpy()[1], g[f"{name}_flow"])


@pytest.mark.gpu
def test_stereo_and_sparse_gpu(torch):
    from paper_1603_03590_b200 import dis_stereo, sparse_correspondences

    g = golden("downscale.npz")
    assert np.array_equal(dis_stereo(g["st3_f1"], g["st3_f2"], stereo_params()), g["st3_flow"])
    for name, dens in (("sp_dense", True), ("sp_chain", False)):
        m = sparse_correspondences(g["sp_f1"], g["sp_f2"], g["sp_seeds"], sparse_params(dens))
        assert np.array_equal(np.array([mm.displacement for mm in m]), g[f"{name}_disp"]), name
        assert np.array_equal(np.array([mm.valid for mm in m]), g[f"{name}_valid"]), name
