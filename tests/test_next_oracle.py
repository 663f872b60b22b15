"""§8(f) "next" rows — pin the C oracle against golden vectors produced by
the reference itself (oracle/gen_golden.py: next_*.npz).  Bit-exact."""

import numpy as np
import pytest

from tests.conftest import golden


def test_compose_flows_oracle(orc):
    g = golden("next_compose.npz")
    for k in range(3):
        assert np.array_equal(orc.compose_flows(g[f"ab{k}"], g[f"bc{k}"]), g[f"out{k}"]), k


def test_compose_shape_mismatch_oracle(orc):
    with pytest.raises(ValueError):
        orc.compose_flows(np.zeros((4, 5, 2)), np.zeros((4, 6, 2)))


def params_from(g):
    """DisParams of a next_*.npz golden (oracle/gen_golden.py _params_dict)."""
    from paper_1603_03590_b200.params import DisParams, VarParams

    outer = int(g["outer"])
    vp = (VarParams(outer_iters_fixed=None if outer < 0 else outer)
          if int(g["variational"]) else None)
    return DisParams(patch_size=int(g["patch_size"]), overlap=float(g["overlap"]),
                     iterations=int(g["iterations"]), finest_scale=int(g["finest"]),
                     coarsest_scale=int(g["coarsest"]),
                     use_mean_normalization=bool(int(g["mean_norm"])),
                     residual_norm=str(g["norm"]), variational=vp, mode=str(g["mode"]),
                     bidirectional=bool(int(g["bidirectional"])))


# ---- stereo (pipeline.py:166-183) ------------------------------------------

@pytest.mark.parametrize("k", range(4))
def test_stereo_end_to_end_oracle(orc, k):
    g = golden(f"next_stereo_{k}.npz")
    flow = orc.dis_stereo(g["f1"], g["f2"], params_from(g))
    assert np.array_equal(flow, g["flow"])
    assert not np.any(flow[..., 1])  # v identically zero


def test_stereo_stages_oracle(orc):
    g = golden("next_stereo_stages.npz")
    r = golden("refine.npz")
    init = r["init"]
    du, dv = orc.sor(init[..., 0], init[..., 1], r["sys"], 1.6, 5, horizontal_only=True)
    assert np.array_equal(du, g["sor_du"]) and np.array_equal(dv, g["sor_dv"])
    from paper_1603_03590_b200.params import VarParams

    lv1 = orc.build_pyramid(r["f1"], 0)[0]
    lv2 = orc.build_pyramid(r["f2"], 0)[0]
    out = orc.refine(init, lv1, lv2, VarParams(), 2, horizontal_only=True)
    assert np.array_equal(out, g["refined_h"])


# ---- bidirectional densification (densification.py:131-153, 194-234) ------

def test_densify_bidirectional_stage_oracle(orc):
    g = golden("next_bidir_stage.npz")
    img1 = orc.build_pyramid(g["f1"], 0)[0][0]
    img2 = orc.build_pyramid(g["f2"], 0)[0][0]
    h, w = img1.shape
    for k in range(3):
        ps, ov = int(g[f"ps{k}"]), float(g[f"ov{k}"])
        xo, _ = orc.axis_origins(w, ps, ov)
        yo, _ = orc.axis_origins(h, ps, ov)
        flow = orc.densify_bidirectional(img1, img2, xo, yo, g[f"fdisp{k}"], g[f"foff{k}"],
                                         xo, yo, g[f"bdisp{k}"], g[f"boff{k}"], ps)
        assert np.array_equal(flow, g[f"flow{k}"]), k


@pytest.mark.parametrize("k", range(4))
def test_bidirectional_end_to_end_oracle(orc, k):
    g = golden(f"next_bidir_{k}.npz")
    p = params_from(g)
    assert p.bidirectional
    assert np.array_equal(orc.dis_flow(g["f1"], g["f2"], p), g["flow"])


# ---- sparse correspondences (pipeline.py:202-287) ---------------------------

SPARSE_CASES = ["dense", "chain", "chain_s0", "dense_bidir"]


def sparse_params(g, name):
    sub = {k[len(name) + 1:]: g[k] for k in g.files if k.startswith(name + "_")
           and not any(k.startswith(o + "_") for o in SPARSE_CASES if o != name and
                       o.startswith(name))}
    import dataclasses

    return dataclasses.replace(params_from(sub), use_densification=bool(int(sub["dens"])))


@pytest.mark.parametrize("name", SPARSE_CASES)
def test_sparse_correspondences_oracle(orc, name):
    g = golden("next_sparse.npz")
    disp, valid = orc.sparse_correspondences(g["f1"], g["f2"], g["seeds"],
                                             sparse_params(g, name))
    assert np.array_equal(valid, g[f"{name}_valid"])
    assert np.array_equal(disp, g[f"{name}_disp"])
