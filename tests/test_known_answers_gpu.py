"""The reference's known-answer cases, restated against this
package's GPU API: pyramid dimensions and gradients, grid spacing and
clamping, densification worked examples, upsampling, refinement and patch
search identities.  Everything runs through the C ABI on the GPU."""

import numpy as np
import pytest

from paper_1603_03590_b200.params import DisParams, VarParams

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    return torch


@pytest.fixture(scope="module")
def st(torch):
    from paper_1603_03590_b200 import stages

    return stages


def _cu(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


# ---- pyramid (core.py:75-128) ------------------------------------------------

def test_pyramid_sintel_level_sizes(torch):
    from paper_1603_03590_b200 import build_pyramid

    pyr = build_pyramid(np.zeros((436, 1024), dtype=np.float32), 5)
    assert [lv.height for lv in pyr.levels] == [436, 218, 109, 54, 27, 13]
    assert [lv.width for lv in pyr.levels] == [1024, 512, 256, 128, 64, 32]


@pytest.mark.parametrize("h,w,coarsest", [(9, 2047, 2), (1080, 1920, 4), (31, 17, 3), (8, 8, 2)])
def test_pyramid_floor_dimension_law(torch, h, w, coarsest):
    from paper_1603_03590_b200 import build_pyramid

    pyr = build_pyramid(np.zeros((h, w)), coarsest)
    for s, lv in enumerate(pyr.levels):
        assert (lv.height, lv.width) == (h >> s, w >> s)


def test_pyramid_refuses_levels_below_two_pixels(torch):
    from paper_1603_03590_b200 import build_pyramid

    with pytest.raises(ValueError):
        build_pyramid(np.zeros((8, 8)), 3)


def test_constant_image_has_zero_gradients_at_every_level(torch):
    from paper_1603_03590_b200 import build_pyramid

    for lv in build_pyramid(np.full((40, 56), 77.0), 3).levels:
        assert not lv.grad_x.any() and not lv.grad_y.any()


def test_linear_ramp_gradients_are_exact(torch):
    from paper_1603_03590_b200 import build_pyramid

    ys, xs = np.mgrid[0:20, 0:32].astype(np.float64)
    lv = build_pyramid(3.0 * xs + 7.0 * ys, 0)[0]
    assert (lv.grad_x.cpu().numpy()[:, 1:-1] == 3.0).all()
    assert (lv.grad_y.cpu().numpy()[1:-1, :] == 7.0).all()


def test_box_mean_of_two_by_two_blocks(torch):
    from paper_1603_03590_b200 import build_pyramid

    block = np.array([[0.0, 2.0, 10.0, 10.0], [4.0, 6.0, 10.0, 10.0]])
    lv1 = build_pyramid(np.vstack([block, block]), 1)[1]
    assert lv1.image.cpu().numpy()[0].tolist() == [3.0, 10.0]


# ---- patch grid (densification.py:50-79) -----------------------------------

@pytest.mark.parametrize("dim,ps,ov,spacing", [(32, 8, 0.0, 8), (32, 8, 0.3, 6),
                                                (32, 8, 0.4, 5), (48, 12, 0.75, 3)])
def test_grid_spacing_floors_the_overlap(torch, st, dim, ps, ov, spacing):
    xo = st.grid_axis(dim, ps, ov)
    assert xo[0] == 0 and xo[1] - xo[0] == spacing
    assert xo[-1] == dim - ps


def test_grid_clamps_the_last_origin(torch, st):
    assert st.grid_axis(17, 8, 0.0).tolist() == [0, 8, 9]
    assert st.grid_axis(16, 8, 0.0).tolist() == [0, 8]


def test_grid_refuses_levels_smaller_than_a_patch(torch, st):
    with pytest.raises(ValueError):
        st.grid_axis(7, 8, 0.0)


# ---- densification (densification.py:110-191) -------------------------------

def _densify(torch, st, ref, qry, ps, ov, disp, offs):
    p = DisParams(patch_size=ps, overlap=ov)
    d = np.asarray(disp, dtype=np.float64)
    u, v = st.densify(_cu(torch, ref[None]), _cu(torch, qry[None]), p, _cu(torch, d[None, :, 0]),
                      _cu(torch, d[None, :, 1]), _cu(torch, np.asarray(offs)[None]))
    return u[0].cpu().numpy(), v[0].cpu().numpy()


def test_densify_single_patch_gives_its_displacement(torch, st):
    u, v = _densify(torch, st, np.zeros((8, 8)), np.full((8, 8), 0.5), 8, 0.0,
                    [[1.25, -0.5]], [0.0])
    assert (u == 1.25).all() and (v == -0.5).all()


def test_densify_two_patch_weighted_average(torch, st):
    # two patches of a 12x8 level (origins x = 0 and 4); at pixel (5, 3) their
    # residuals are 1 and 4 -> weights 1 and 1/4 for u = 1 and u = 3
    qry = np.zeros((8, 12))
    qry[3, 6] = 1.0
    qry[3, 8] = 4.0
    u, v = _densify(torch, st, np.zeros((8, 12)), qry, 8, 0.5, [[1.0, 0.0], [3.0, 0.0]],
                    [0.0, 0.0])
    assert u[3, 5] == pytest.approx((1.0 * 1.0 + 0.25 * 3.0) / 1.25, abs=1e-12)
    assert v[3, 5] == 0.0


def test_densify_shared_displacement_is_exact(torch, st):
    rng = np.random.default_rng(13)
    ref = rng.uniform(0, 255, (14, 20))
    qry = rng.uniform(0, 255, (14, 20))
    n = len(st.grid_axis(20, 8, 0.5)) * len(st.grid_axis(14, 8, 0.5))
    u, v = _densify(torch, st, ref, qry, 8, 0.5, np.tile([2.5, -1.0], (n, 1)), np.zeros(n))
    assert np.abs(u - 2.5).max() <= 1e-12 and np.abs(v + 1.0).max() <= 1e-12


def test_densify_is_convex_and_covers_random_layouts(torch, st):
    rng = np.random.default_rng(14)
    for _ in range(10):
        ps = int(rng.integers(4, 10))
        w, h = int(rng.integers(ps, 40)), int(rng.integers(ps, 40))
        ov = float(rng.uniform(0, 0.9))
        n = len(st.grid_axis(w, ps, ov)) * len(st.grid_axis(h, ps, ov))
        disp = rng.normal(0, 2, (n, 2))
        u, v = _densify(torch, st, rng.uniform(0, 255, (h, w)), rng.uniform(0, 255, (h, w)), ps,
                        ov, disp, rng.normal(0, 1, n))
        for comp, c in ((u, 0), (v, 1)):
            assert comp.min() >= disp[:, c].min() - 1e-12
            assert comp.max() <= disp[:, c].max() + 1e-12


# ---- upsampling (core.py:154-190) -------------------------------------------

def test_upsample_constant_field_doubles_exactly(torch, st):
    u = _cu(torch, np.full((1, 13, 17), 1.75))
    v = _cu(torch, np.full((1, 13, 17), -0.5))
    ou, ov = st.upsample_flow(u, v, 34, 27)
    assert (ou.cpu().numpy() == 3.5).all() and (ov.cpu().numpy() == -1.0).all()


def test_compose_with_zero_first_field_returns_the_second(torch):
    from paper_1603_03590_b200 import compose_flows

    bc = np.random.default_rng(3).normal(0, 3, (9, 11, 2))
    assert np.array_equal(compose_flows(np.zeros_like(bc), bc), bc)


# ---- refinement (variational.py:220-275) ------------------------------------

def test_refine_on_constant_images_is_the_identity(torch, st):
    lv = st.build_pyramid(np.full((20, 26), 64.0), 0)[0]
    fu = _cu(torch, np.full((1, 20, 26), 3.25))
    fv = _cu(torch, np.full((1, 20, 26), -1.5))
    u, v = st.refine(fu, fv, lv, lv, DisParams(variational=VarParams()), 3)
    assert (u.cpu().numpy() == 3.25).all() and (v.cpu().numpy() == -1.5).all()


# ---- patch search (inverse_search.py:113-189) -------------------------------

def test_patch_search_on_identical_frames_stays_at_zero(torch, st):
    img = np.random.default_rng(21).uniform(0, 255, (32, 48))
    lv = st.build_pyramid(img, 0)[0]
    out = st.patch_search(lv, lv["img"], DisParams(patch_size=8, overlap=0.5, iterations=16))
    assert not out["u"].any() and not out["v"].any()
    assert not out["off"].any() and not out["mar"].any()


def test_constant_patches_are_invalid_and_keep_their_init(torch, st):
    lv = st.build_pyramid(np.full((24, 24), 9.0), 0)[0]
    q = st.build_pyramid(np.random.default_rng(2).uniform(0, 255, (24, 24)), 0)[0]
    coarse = _cu(torch, np.full((1, 12, 12), 0.75))
    out = st.patch_search(lv, q["img"], DisParams(patch_size=8, overlap=0.0, iterations=8),
                          coarse, coarse)
    assert not out["valid"].any()
    assert (out["u"].cpu().numpy() == 1.5).all() and (out["v"].cpu().numpy() == 1.5).all()


# ---- reference test intents on a rendered texture (test_inverse_search.py,
# test_variational.py), through the grid stage API ---------------------------

def _waves(seed, n=8, lo=6.0, hi=20.0):
    rng = np.random.default_rng(seed)
    lam = rng.uniform(lo, hi, n)
    ang = rng.uniform(0, 2 * np.pi, n)
    ph = rng.uniform(0, 2 * np.pi, n)
    amp = rng.uniform(10.0, 30.0, n)
    return lam, ang, ph, amp


def _render(w, width, height, shift=(0.0, 0.0)):
    """sum of plane waves sampled at (x - sx, y - sy): a continuous texture
    translated by `shift` (so the flow from the unshifted frame is `shift`)."""
    lam, ang, ph, amp = w
    ys, xs = np.mgrid[0:height, 0:width].astype(np.float64)
    xs = xs - shift[0]
    ys = ys - shift[1]
    img = np.full((height, width), 128.0)
    for L, a, p, A in zip(lam, ang, ph, amp):
        img += A * np.sin(2 * np.pi * (np.cos(a) * xs + np.sin(a) * ys) / L + p)
    return img


def _search_center(st, ref_img, qry_img, **kw):
    """The 8px patch centred at (16, 16) of a 32x32 level (grid spacing 4,
    origin (12, 12), patch index 3 * 7 + 3); returns (u, v, mar)."""
    ref = st.build_pyramid(ref_img, 0)[0]
    qry = st.build_pyramid(qry_img, 0)[0]
    p = DisParams(patch_size=8, overlap=0.5, **kw)
    out = st.patch_search(ref, qry["img"], p)
    i = 3 * 7 + 3
    return (float(out["u"][0, i]), float(out["v"][0, i]), float(out["mar"][0, i]))


def test_identity_is_an_exact_fixed_point(torch, st):
    img = _render(_waves(4), 32, 32)
    u, v, mar = _search_center(st, img, img, iterations=16)
    assert u == 0.0 and v == 0.0 and mar == 0.0


def test_integer_translation_is_recovered(torch, st):
    w = _waves(5)
    u, v, _ = _search_center(st, _render(w, 32, 32), _render(w, 32, 32, (2.0, 1.0)),
                             iterations=16)
    assert abs(u - 2.0) < 0.05 and abs(v - 1.0) < 0.05


def test_large_translation_is_outside_the_single_level_basin(torch, st):
    w = _waves(6)
    ref = st.build_pyramid(_render(w, 64, 32), 0)[0]
    qry = st.build_pyramid(_render(w, 64, 32, (20.0, 0.0)), 0)[0]
    out = st.patch_search(ref, qry["img"], DisParams(patch_size=8, overlap=0.5, iterations=16))
    i = 3 * 15 + 7  # centre (32, 16) of a 15 x 7 grid
    err = np.hypot(float(out["u"][0, i]) - 20.0, float(out["v"][0, i]))
    assert err > 1.0


def test_mean_normalization_ignores_a_constant_offset(torch, st):
    w = _waves(8)
    ref = _render(w, 32, 32)
    qry = _render(w, 32, 32, (1.3, -0.7))
    a = _search_center(st, ref, qry, iterations=12)
    b = _search_center(st, ref, qry + 50.0, iterations=12)
    assert abs(a[0] - b[0]) <= 1e-9 and abs(a[1] - b[1]) <= 1e-9
    c = _search_center(st, ref, qry + 50.0, iterations=12, use_mean_normalization=False)
    assert np.hypot(c[0] - a[0], c[1] - a[1]) > 0.01


def test_patch_search_is_deterministic(torch, st):
    w = _waves(9)
    ref, qry = _render(w, 32, 32), _render(w, 32, 32, (1.5, 0.5))
    assert _search_center(st, ref, qry, iterations=12) == _search_center(st, ref, qry,
                                                                         iterations=12)


def test_huber_norm_reduces_outlier_influence(torch, st):
    w = _waves(10)
    ref = _render(w, 32, 32)
    qry = _render(w, 32, 32, (1.0, 0.5))
    qry[12:16, 12:16] += 200.0  # corrupt part of the window
    l2 = _search_center(st, ref, qry, iterations=12)
    hub = _search_center(st, ref, qry, iterations=12, residual_norm="huber", huber_b=1.0)
    assert np.hypot(hub[0] - 1.0, hub[1] - 0.5) < np.hypot(l2[0] - 1.0, l2[1] - 0.5)


def test_refine_reduces_the_error_of_a_noisy_initialisation(torch, st):
    w = _waves(11, lo=8.0, hi=24.0)
    H, W = 40, 48
    ref = st.build_pyramid(_render(w, W, H), 0)[0]
    qry = st.build_pyramid(_render(w, W, H, (1.0, -0.5)), 0)[0]
    rng = np.random.default_rng(12)
    u0 = 1.0 + rng.normal(0, 0.3, (1, H, W))
    v0 = -0.5 + rng.normal(0, 0.3, (1, H, W))
    u, v = st.refine(_cu(torch, u0), _cu(torch, v0), ref, qry,
                     DisParams(variational=VarParams()), 3)
    inner = (slice(None), slice(4, H - 4), slice(4, W - 4))
    e0 = np.hypot(u0 - 1.0, v0 + 0.5)[inner].mean()
    e1 = np.hypot(u.cpu().numpy() - 1.0, v.cpu().numpy() + 0.5)[inner].mean()
    assert e1 < 0.5 * e0


def test_refine_horizontal_only_keeps_v(torch, st):
    w = _waves(13)
    ref = st.build_pyramid(_render(w, 40, 24), 0)[0]
    qry = st.build_pyramid(_render(w, 40, 24, (1.5, 0.0)), 0)[0]
    rng = np.random.default_rng(14)
    u0 = _cu(torch, rng.normal(1.5, 0.2, (1, 24, 40)))
    v0 = torch.zeros_like(u0)
    u, v = st.refine(u0, v0, ref, qry, DisParams(mode="stereo", variational=VarParams()), 2)
    assert not v.any()
    assert not torch.equal(u, u0)


def test_refine_rejects_non_finite_flow(torch, st):
    lv = st.build_pyramid(np.random.default_rng(15).uniform(0, 255, (16, 16)), 0)[0]
    u0 = torch.zeros((1, 16, 16), dtype=torch.float64, device="cuda")
    u0[0, 8, 8] = float("nan")
    with pytest.raises(RuntimeError):
        st.refine(u0, torch.zeros_like(u0), lv, lv, DisParams(variational=VarParams()), 1)


def test_ramp_patch_is_invalid_and_checkerboard_valid(torch, st):
    # test_inverse_search.py:36-55 intent, through the grid stage: a unit
    # horizontal ramp gives a singular Hessian (invalid, keeps its init), a
    # checkerboard a well-conditioned one (valid)
    ys, xs = np.mgrid[0:24, 0:24].astype(np.float64)
    ramp = st.build_pyramid(xs * 1.0, 0)[0]
    out = st.patch_search(ramp, ramp["img"], DisParams(patch_size=8, overlap=0.0, iterations=4))
    assert not out["valid"].any()
    checker = 100.0 * (((xs // 2) + (ys // 2)) % 2) + 20.0
    lv = st.build_pyramid(checker, 0)[0]
    out = st.patch_search(lv, lv["img"], DisParams(patch_size=8, overlap=0.0, iterations=4))
    assert out["valid"].all()


def test_refine_barely_moves_the_exact_solution(torch, st):
    # test_variational.py:74-81 intent: at the true translation the update
    # stays small
    w = _waves(16, lo=8.0, hi=24.0)
    H, W = 40, 48
    ref = st.build_pyramid(_render(w, W, H), 0)[0]
    qry = st.build_pyramid(_render(w, W, H, (0.75, -0.5)), 0)[0]
    u0 = np.full((1, H, W), 0.75)
    v0 = np.full((1, H, W), -0.5)
    u, v = st.refine(_cu(torch, u0), _cu(torch, v0), ref, qry,
                     DisParams(variational=VarParams()), 1)
    inner = (slice(None), slice(4, H - 4), slice(4, W - 4))
    drift = np.hypot(u.cpu().numpy() - 0.75, v.cpu().numpy() + 0.5)[inner].mean()
    assert drift < 0.05


def test_more_outer_iterations_lower_the_error(torch, st):
    # test_variational.py:120-131 intent
    w = _waves(17, lo=8.0, hi=24.0)
    H, W = 40, 48
    ref = st.build_pyramid(_render(w, W, H), 0)[0]
    qry = st.build_pyramid(_render(w, W, H, (1.0, 0.5)), 0)[0]
    rng = np.random.default_rng(18)
    u0 = _cu(torch, 1.0 + rng.normal(0, 0.4, (1, H, W)))
    v0 = _cu(torch, 0.5 + rng.normal(0, 0.4, (1, H, W)))
    inner = (slice(None), slice(4, H - 4), slice(4, W - 4))
    errs = []
    for outer in (1, 4):
        u, v = st.refine(u0, v0, ref, qry, DisParams(variational=VarParams()), outer)
        errs.append(np.hypot(u.cpu().numpy() - 1.0, v.cpu().numpy() - 0.5)[inner].mean())
    assert errs[1] < errs[0]


def _ssd_meannorm(ref, qry, x0, y0, ps, u, v):
    """mean-normalised SSD of the ps x ps window at (x0, y0) against the query
    sampled at +(u, v) (clamped bilinear, an independent restatement)."""
    h, w = qry.shape
    ys, xs = np.mgrid[0:ps, 0:ps].astype(np.float64)
    x = np.clip(x0 + xs + u, 0.0, w - 1.0)
    y = np.clip(y0 + ys + v, 0.0, h - 1.0)
    xi = np.floor(x).astype(int)
    yi = np.floor(y).astype(int)
    x1 = np.minimum(xi + 1, w - 1)
    y1 = np.minimum(yi + 1, h - 1)
    fx, fy = x - xi, y - yi
    a = qry[yi, xi] + fx * (qry[yi, x1] - qry[yi, xi])
    b = qry[y1, xi] + fx * (qry[y1, x1] - qry[y1, xi])
    warped = a + fy * (b - a)
    t = ref[y0:y0 + ps, x0:x0 + ps]
    d = (warped - warped.mean()) - (t - t.mean())
    return float((d * d).sum())


def test_first_gauss_newton_step_reduces_the_ssd(torch, st):
    # test_inverse_search.py:106-125 intent: one iteration from zero lowers the
    # (mean-normalised) SSD for >= 99 % of valid patches under small shifts
    rng = np.random.default_rng(7)
    n = 300
    refs, qrys = [], []
    for _ in range(n):
        w = _waves(int(rng.integers(1 << 30)), n=6, lo=16.0, hi=48.0)
        a = rng.uniform(0, 2 * np.pi)
        r = rng.uniform(0.25, 1.0)
        refs.append(_render(w, 24, 24))
        qrys.append(_render(w, 24, 24, (r * np.cos(a), r * np.sin(a))))
    ref_b, qry_b = np.stack(refs), np.stack(qrys)
    lr = st.build_pyramid(ref_b, 0)[0]
    lq = st.build_pyramid(qry_b, 0)[0]
    out = st.patch_search(lr, lq["img"], DisParams(patch_size=8, overlap=0.5, iterations=1))
    i = 2 * 5 + 2  # the patch at origin (8, 8) of a 5 x 5 grid
    u = out["u"][:, i].cpu().numpy()
    v = out["v"][:, i].cpu().numpy()
    valid = out["valid"][:, i].cpu().numpy().astype(bool)
    reduced = checked = 0
    for k in range(n):
        if not valid[k]:
            continue
        checked += 1
        if _ssd_meannorm(ref_b[k], qry_b[k], 8, 8, 8, u[k], v[k]) < \
                _ssd_meannorm(ref_b[k], qry_b[k], 8, 8, 8, 0.0, 0.0):
            reduced += 1
    assert checked >= 0.8 * n
    assert reduced >= 0.99 * checked
