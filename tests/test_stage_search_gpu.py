"""The reference-signature inverse-search stage functions (inverse_search.py:
283-494: PatchSet, precompute_patch_set, optimize_patch_set,
refresh_patch_stats, PatchState, precompute_patch, optimize_patch) and the
densification module's init_patches / reset_outliers on the GPU
(csrc/stage_search.cu through the C ABI) against the reference's own outputs
(oracle/gen_golden.py gen_stage_search -> tests/golden/stage_search.npz):
real (non-grid) window origins, ps 8 and 12, flow and horizontal-only
conditioning, L2 / L1 / Huber with and without mean normalisation.
Tolerance 0 (np.array_equal)."""

import numpy as np
import pytest

from tests.conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def levels():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    from paper_1603_03590_b200 import build_pyramid

    g = golden("stage_search.npz")
    return g, build_pyramid(g["f1"], 0)[0], build_pyramid(g["f2"], 0)[0]


@pytest.mark.parametrize("ps,hz", [(8, False), (8, True), (12, False), (12, True)])
def test_precompute_patch_set(levels, ps, hz):
    from paper_1603_03590_b200 import precompute_patch_set

    g, l1, _ = levels
    p = precompute_patch_set(l1, g["xs"], g["ys"], ps, horizontal_only=hz)
    tag = f"ps{ps}_{'h' if hz else 'f'}"
    assert np.array_equal(p.templates, g[f"{tag}_tmpl"])
    assert np.array_equal(p.steep_x, g[f"{tag}_sdx"])
    assert np.array_equal(p.steep_y, g[f"{tag}_sdy"])
    assert np.array_equal(p.hessian, g[f"{tag}_hess"])
    assert np.array_equal(p.hessian_inv, g[f"{tag}_hinv"])
    assert np.array_equal(p.template_mean, g[f"{tag}_mean"])
    assert np.array_equal(p.valid, g[f"{tag}_valid"])
    assert len(p) == len(g["xs"])


@pytest.mark.parametrize("norm", ["l2", "l1", "huber"])
@pytest.mark.parametrize("mn", [True, False])
def test_optimize_patch_set(levels, norm, mn):
    from paper_1603_03590_b200 import optimize_patch_set, precompute_patch_set

    g, l1, l2 = levels
    p = precompute_patch_set(l1, g["xs"], g["ys"], 8)
    p.init_displacement = g["init"].copy()
    optimize_patch_set(p, l2, 24, residual_norm=norm, huber_b=2.0, mean_normalization=mn)
    tag = f"opt_{norm}_{int(mn)}"
    assert np.array_equal(p.displacement, g[f"{tag}_disp"])
    assert np.array_equal(p.offset, g[f"{tag}_off"])
    assert np.array_equal(p.mean_abs_residual, g[f"{tag}_mar"])


def test_reset_and_refresh_patch_stats(levels):
    from paper_1603_03590_b200 import (optimize_patch_set, precompute_patch_set,
                                       refresh_patch_stats, reset_outliers)

    g, l1, l2 = levels
    p = precompute_patch_set(l1, g["xs"], g["ys"], 8)
    p.init_displacement = g["init"].copy()
    optimize_patch_set(p, l2, 24, residual_norm="l2", huber_b=2.0, mean_normalization=True)
    kept = reset_outliers(p.displacement, g["init"], 8)
    assert np.array_equal(kept, g["refresh_disp"])
    p.displacement = kept
    refresh_patch_stats(p, l2, g["refresh_sel"], True)
    assert np.array_equal(p.offset, g["refresh_off"])
    assert np.array_equal(p.mean_abs_residual, g["refresh_mar"])
    before = p.offset.copy()
    refresh_patch_stats(p, l2, np.zeros(len(p), dtype=bool))  # nothing selected: untouched
    assert np.array_equal(p.offset, before)


def test_single_patch_interface(levels):
    import dataclasses

    from paper_1603_03590_b200 import optimize_patch, precompute_patch

    g, l1, l2 = levels
    st = precompute_patch(l1, (70.3, 40.8), 8)
    assert np.array_equal(st.template, g["single_tmpl"])
    assert np.array_equal(st.steepest_descent, g["single_sd"])
    assert np.array_equal(st.hessian_inverse, g["single_hinv"])
    st = dataclasses.replace(st, init_displacement=np.array([1.25, -0.5]))
    out = optimize_patch(st, l2, 32, residual_norm="huber", huber_b=1.5)
    assert np.array_equal(out.displacement, g["single_disp"])
    assert out.mean_offset == float(g["single_off"])
    assert out.mean_abs_residual == float(g["single_mar"])
    with pytest.raises(ValueError):
        optimize_patch(st, l2, 4, residual_norm="l3")


def test_reference_known_answers(levels):
    """The reference's own known answers (pkg/tests/test_inverse_search.py:
    28-76): a constant patch is invalid with H = 0; a unit ramp has
    H = [[64, 0], [0, 0]] and is invalid; the template is the image itself at
    integer coordinates; identity displacement is exactly (0, 0) with zero
    residual."""
    import torch

    from paper_1603_03590_b200 import PyramidLevel, optimize_patch, precompute_patch

    def level(img):
        gx = np.zeros_like(img)
        gy = np.zeros_like(img)
        gx[:, 1:-1] = 0.5 * (img[:, 2:] - img[:, :-2])
        gx[:, 0] = 0.5 * (img[:, 1] - img[:, 0])
        gx[:, -1] = 0.5 * (img[:, -1] - img[:, -2])
        gy[1:-1] = 0.5 * (img[2:] - img[:-2])
        gy[0] = 0.5 * (img[1] - img[0])
        gy[-1] = 0.5 * (img[-1] - img[-2])
        t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
        return PyramidLevel(t(img), t(gx), t(gy), 0)

    const = level(np.full((16, 16), 7.0))
    st = precompute_patch(const, (8.0, 8.0), 8)
    assert not st.valid and st.hessian_inverse is None and not st.hessian.any()
    ramp = level(np.tile(np.arange(16.0), (16, 1)))
    st = precompute_patch(ramp, (8.0, 8.0), 8)
    assert np.array_equal(st.hessian, np.array([[64.0, 0.0], [0.0, 0.0]])) and not st.valid
    g, l1, l2 = levels
    img = l1.image.cpu().numpy()
    st = precompute_patch(l1, (8.0, 8.0), 8)
    assert np.array_equal(st.template, img[4:12, 4:12])
    same = optimize_patch(st, l1, 16)
    assert np.array_equal(same.displacement, [0.0, 0.0]) and same.mean_abs_residual == 0.0
