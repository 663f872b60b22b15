"""Pin the C oracle (oracle/dis_oracle.c) against golden vectors produced by
the reference itself (oracle/gen_golden.py).  Everything is bit-exact."""

import numpy as np
import pytest

from paper_1603_03590_b200.params import DisParams, VarParams
from tests.conftest import golden


def test_pyramid_levels_bit_exact(orc):
    g = golden("pyramid.npz")
    levels = orc.build_pyramid(g["img"], 4)
    for s, (img, gx, gy) in enumerate(levels):
        assert np.array_equal(img, g[f"L{s}_img"]), s
        assert np.array_equal(gx, g[f"L{s}_gx"]), s
        assert np.array_equal(gy, g[f"L{s}_gy"]), s
        dd = np.stack(orc.second_derivatives(gx, gy))
        assert np.array_equal(dd, g[f"L{s}_dd"]), s


def test_box_mean_order_80k_blocks(orc):
    g = golden("pyramid.npz")
    big = np.random.default_rng(1000).uniform(0, 255, size=(200, 400))
    assert np.array_equal(orc.box_downsample(big), g["box_out"])


def test_bilinear_forms(orc):
    g = golden("samplers.npz")
    assert np.array_equal(orc.bilinear_map(g["bm_img"], g["bm_x"], g["bm_y"]), g["bm_np"])
    img = np.ascontiguousarray(g["bm_img"])
    nb = np.array([orc.lib().orc_bilin_nb(img.ctypes.data_as(orc._D), img.shape[0],
                                          img.shape[1], float(x), float(y))
                   for x, y in zip(g["bm_x"], g["bm_y"])])
    assert np.array_equal(nb, g["bm_nb"])


def test_upsample(orc):
    g = golden("samplers.npz")
    assert np.array_equal(orc.upsample(g["flow"], 35, 27), g["up_27x35"])
    assert np.array_equal(orc.upsample(g["flow"], 34, 26), g["up_26x34"])


def test_grids(orc):
    g = golden("samplers.npz")
    off = 0
    for dim, ps, ov, sp, cnt in zip(g["grid_dims"], g["grid_ps"], g["grid_ov"],
                                    g["grid_spacing"], g["grid_counts"]):
        o, spacing = orc.axis_origins(int(dim), int(ps), float(ov))
        assert spacing == sp
        assert np.array_equal(o, g["grid_origins"][off:off + cnt])
        off += cnt


@pytest.mark.parametrize("name,s,ps,ov,iters,norm", [
    ("search_c1_like.npz", 1, 8, 0.5, 32, 0),
    ("search_c2_like.npz", 0, 12, 0.75, 128, 0),
    ("search_huber.npz", 0, 8, 0.3, 16, 2),
    ("search_l1.npz", 0, 8, 0.3, 16, 1),
])
def test_patch_search_and_densify(orc, name, s, ps, ov, iters, norm):
    g = golden(name)
    lv1 = orc.build_pyramid(g["in_f1"], s)[s]
    lv2 = orc.build_pyramid(g["in_f2"], s)[s]
    xo, _ = orc.axis_origins(lv1[0].shape[1], ps, ov)
    yo, _ = orc.axis_origins(lv1[0].shape[0], ps, ov)
    assert np.array_equal(xo, g["x_origins"]) and np.array_equal(yo, g["y_origins"])
    coarse = g["in_coarse"] if "in_coarse" in g.files else None
    init = orc.init_patches(xo, yo, ps, coarse)
    assert np.array_equal(init, g["init"])
    r = orc.patch_search(lv1[0], lv1[1], lv1[2], lv2[0], xo, yo, ps, init, iters,
                         norm_code=norm, huber_b=1.0)
    assert np.array_equal(r["valid"], g["valid"])
    assert np.array_equal(r["hinv"], g["hinv"])
    assert np.array_equal(r["mean_t"], g["mean_t"])
    assert np.array_equal(r["raw_disp"], g["raw_disp"])
    assert np.array_equal(r["reset"], g["reset"])
    assert np.array_equal(r["disp"], g["disp"])
    assert np.array_equal(r["offset"], g["off"])
    assert np.array_equal(r["mar"], g["mar"])
    dense = orc.densify(lv1[0], lv2[0], xo, yo, ps, r["disp"], r["offset"])
    assert np.array_equal(dense, g["dense"])


def test_refine(orc):
    g = golden("refine.npz")
    lv1 = orc.build_pyramid(g["f1"], 0)[0]
    lv2 = orc.build_pyramid(g["f2"], 0)[0]
    vp = VarParams()
    assert np.array_equal(orc.refine(g["init"], lv1, lv2, vp, 1), g["refined_s0"])
    assert np.array_equal(orc.refine(g["init"], lv1, lv2, vp, 3), g["refined_s2"])
    assert np.array_equal(orc.refine(g["init"], lv1, lv2, vp, 1), g["refined_fixed1"])


def _params_from(g):
    outer = int(g["outer"])
    return DisParams(
        patch_size=int(g["patch_size"]), overlap=float(g["overlap"]),
        iterations=int(g["iterations"]), finest_scale=int(g["finest"]),
        coarsest_scale=int(g["coarsest"]),
        variational=VarParams(outer_iters_fixed=None if outer < 0 else outer))


@pytest.mark.parametrize("case", ["c0", "c0_default_outer", "c1", "c2", "c3", "c4"])
def test_end_to_end_small(orc, case):
    g = golden(f"e2e_{case}.npz")
    flow = orc.dis_flow(g["f1"], g["f2"], _params_from(g))
    assert np.array_equal(flow, g["flow"])
