"""The reference-signature stage functions (paper_1603_03590_b200.densification,
.variational, image_gradients, upsample_flow) against the reference's own
outputs (tests/golden).  The grid axes come from the library's host grid
code (CPU test); init, reset, densification, refinement, gradients and
upsampling run on the GPU.  Bit-exact."""

import numpy as np
import pytest

from paper_1603_03590_b200.params import VarParams
from tests.conftest import golden

gpu = pytest.mark.gpu


def test_create_grid_matches_reference_grids():
    from paper_1603_03590_b200 import create_grid

    g = golden("samplers.npz")
    off = 0
    for dim, ps, ov, sp, n in zip(g["grid_dims"], g["grid_ps"], g["grid_ov"],
                                  g["grid_spacing"], g["grid_counts"]):
        grid = create_grid(int(dim), int(ps), int(ps), float(ov))
        assert grid.spacing == sp
        assert np.array_equal(grid.x_origins, g["grid_origins"][off:off + n])
        off += n
    with pytest.raises(ValueError):
        create_grid(7, 16, 8, 0.0)
    with pytest.raises(ValueError):
        create_grid(16, 16, 8, 1.0)


@gpu
def test_init_patches_and_reset_outliers_match_reference():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    from paper_1603_03590_b200 import create_grid, init_patches, reset_outliers

    g = golden("search_c1_like.npz")
    grid = create_grid(128, 54, 8, 0.5)
    assert np.array_equal(grid.x_origins, g["x_origins"])
    init = init_patches(grid, g["in_coarse"], 2)
    assert np.array_equal(init, g["init"])
    assert np.array_equal(reset_outliers(g["raw_disp"], init, 8), g["disp"])
    assert not init_patches(grid, None, 2).any()


@gpu
def test_image_gradients_and_upsample_flow(orc):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    from paper_1603_03590_b200 import image_gradients, upsample_flow

    p = golden("pyramid.npz")
    gx, gy = image_gradients(p["img"])
    assert np.array_equal(gx, p["L0_gx"]) and np.array_equal(gy, p["L0_gy"])
    s = golden("samplers.npz")
    assert np.array_equal(upsample_flow(s["flow"], 35, 27, 2), s["up_27x35"])
    assert np.array_equal(upsample_flow(s["flow"], 34, 26, 2), s["up_26x34"])


@gpu
def test_densify_and_bidirectional_match_reference(orc):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    from paper_1603_03590_b200 import create_grid, densify, densify_bidirectional

    g = golden("search_c1_like.npz")
    ref = orc.build_pyramid(g["in_f1"], 1)[1][0]
    qry = orc.build_pyramid(g["in_f2"], 1)[1][0]
    grid = create_grid(128, 54, 8, 0.5)
    assert np.array_equal(densify(grid, g["disp"], g["off"], ref, qry), g["dense"])
    b = golden("next_bidir_stage.npz")
    r0 = orc.build_pyramid(b["f1"], 0)[0][0]
    q0 = orc.build_pyramid(b["f2"], 0)[0][0]
    for k in range(3):
        gr = create_grid(128, 54, int(b[f"ps{k}"]), float(b[f"ov{k}"]))
        got = densify_bidirectional(gr, b[f"fdisp{k}"], b[f"foff{k}"], gr, b[f"bdisp{k}"],
                                    b[f"boff{k}"], r0, q0)
        assert np.array_equal(got, b[f"flow{k}"]), k


@gpu
def test_refine_matches_reference(orc):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    from paper_1603_03590_b200 import PyramidLevel, refine

    r = golden("refine.npz")

    def level(f):
        img, gx, gy = orc.build_pyramid(f, 0)[0]
        return PyramidLevel(img, gx, gy, 0)

    l1, l2 = level(r["f1"]), level(r["f2"])
    assert np.array_equal(refine(r["init"], l1, l2, VarParams(), 0), r["refined_s0"])
    assert np.array_equal(refine(r["init"], l1, l2, VarParams(), 2), r["refined_s2"])
    assert np.array_equal(refine(r["init"], l1, l2, VarParams(outer_iters_fixed=1), 4),
                          r["refined_fixed1"])
    h = golden("next_stereo_stages.npz")
    assert np.array_equal(refine(r["init"], l1, l2, VarParams(outer_iters_fixed=2), 0,
                                 horizontal_only=True), h["refined_h"])
    with pytest.raises(ValueError):
        bad = r["init"].copy()
        bad[0, 0, 0] = np.nan
        refine(bad, l1, l2, VarParams(), 0)
