"""Generate golden vectors by running the REFERENCE itself (test infra).

Run in the build container only (needs /root/reference):

    python oracle/gen_golden.py

Writes tests/golden/*.npz.  Imports the reference package from
/root/reference/pkg/src with NUMBA_CACHE_DIR redirected to /tmp so nothing
is written into the read-only reference tree.  Every array stored here is a
reference output on a seeded input; tests/test_oracle_golden.py checks the C
oracle against them bit-for-bit and tests/test_gpu_parity.py checks the CUDA
path against the oracle (and the goldens) on the GPU box.

Versions recorded in every file: numpy, numba, scipy, python.
"""

from __future__ import annotations

import dataclasses
import hashlib
import os
import platform
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import disflow  # noqa: E402  (the reference)
from disflow import core, densification, inverse_search, pipeline, variational  # noqa: E402

from tools import synth  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")


@dataclasses.dataclass(frozen=True)
class VarParamsFixed(core.VarParams):
    """Reference-side outer-iteration override."""

    fixed_outer: int = 1

    def outer_iters(self, scale_index: int) -> int:
        return self.fixed_outer


def versions():
    import numba
    import scipy

    return dict(numpy=np.__version__, numba=numba.__version__, scipy=scipy.__version__,
                python=platform.python_version())


def ref_params(cfg, outer_fixed=1, coarsest=None):
    vp = (VarParamsFixed(fixed_outer=outer_fixed) if outer_fixed is not None
          else core.VarParams())
    return core.DisParams(
        patch_size=cfg.patch_size, overlap=cfg.overlap, iterations=cfg.iterations,
        finest_scale=cfg.finest_scale,
        coarsest_scale=cfg.coarsest_scale if coarsest is None else coarsest,
        variational=vp)


def save(name, **arrays):
    meta = versions()
    np.savez_compressed(os.path.join(OUT, name), **arrays,
                        **{f"meta_{k}": np.array(v) for k, v in meta.items()})
    print("wrote", name, sorted(arrays))


def gen_pyramid():
    rng = np.random.default_rng(100)
    img = rng.uniform(0, 255, size=(91, 133)).astype(np.float32)
    pyr = core.build_pyramid(img, 4)
    d = {"img": img}
    for s, lvl in enumerate(pyr.levels):
        d[f"L{s}_img"] = lvl.image
        d[f"L{s}_gx"] = lvl.grad_x
        d[f"L{s}_gy"] = lvl.grad_y
        gxx, gxy, gyx, gyy = variational._second_derivatives(lvl)
        d[f"L{s}_dd"] = np.stack([gxx, gxy, gyx, gyy])
    # the 10^6-block box-mean order check (core.py:88-98)
    # regenerate in the test with default_rng(1000).uniform(0, 255, (200, 400))
    big = np.random.default_rng(1000).uniform(0, 255, size=(200, 400))
    d["box_out"] = core._box_downsample(big, 2)
    save("pyramid.npz", **d)


def gen_samplers():
    rng = np.random.default_rng(101)
    flow = rng.normal(0, 3, size=(13, 17, 2))
    d = {"flow": flow}
    d["up_27x35"] = core.upsample_flow(flow, 35, 27, 2)
    d["up_26x34"] = core.upsample_flow(flow, 34, 26, 2)
    img = rng.uniform(0, 255, size=(11, 9))
    xs = rng.uniform(-3, 12, size=500)
    ys = rng.uniform(-3, 14, size=500)
    d["bm_img"] = img
    d["bm_x"] = xs
    d["bm_y"] = ys
    d["bm_np"] = core.bilinear_map(img, xs, ys)
    d["bm_nb"] = np.array([inverse_search._bilin(img, x, y) for x, y in zip(xs, ys)])
    # grids
    grids = []
    for (dim, ps, ov) in [(1024, 8, 0.3), (436, 8, 0.5), (436, 12, 0.75), (17, 8, 0.0),
                          (12, 8, 0.999), (54, 8, 0.4), (13, 8, 0.3), (1080, 8, 0.5),
                          (2160, 12, 0.75), (33, 5, 0.37)]:
        g = densification.create_grid(dim, ps, ps, ov)
        grids.append((dim, ps, ov, g.spacing, g.x_origins))
    d["grid_dims"] = np.array([g[0] for g in grids])
    d["grid_ps"] = np.array([g[1] for g in grids])
    d["grid_ov"] = np.array([g[2] for g in grids])
    d["grid_spacing"] = np.array([g[3] for g in grids])
    d["grid_origins"] = np.concatenate([g[4] for g in grids])
    d["grid_counts"] = np.array([len(g[4]) for g in grids])
    save("samplers.npz", **d)


def search_case(f1, f2, s, ps, ov, iters, coarse_flow, norm="l2", mean_norm=True):
    """Replicates pipeline._ScaleState.search (pipeline.py:54-82) on level s
    and returns its outputs."""
    pyr1 = core.build_pyramid(f1, s)
    pyr2 = core.build_pyramid(f2, s)
    ref, qry = pyr1[s], pyr2[s]
    grid = densification.create_grid(ref.width, ref.height, ps, ov)
    u_init = densification.init_patches(grid, coarse_flow, 2)
    starts = grid.starts
    pset = inverse_search.precompute_patch_set(ref, starts[:, 0], starts[:, 1], ps)
    pset.init_displacement = u_init
    inverse_search.optimize_patch_set(pset, qry, iters, residual_norm=norm,
                                      mean_normalization=mean_norm)
    raw = pset.displacement.copy()
    raw_off = pset.offset.copy()
    kept = densification.reset_outliers(pset.displacement, u_init, ps)
    was_reset = (kept != pset.displacement).any(axis=1)
    pset.displacement = kept
    inverse_search.refresh_patch_stats(pset, qry, was_reset, mean_norm)
    flow = densification.densify(grid, pset.displacement, pset.offset, ref.image, qry.image)
    return dict(x_origins=grid.x_origins, y_origins=grid.y_origins, init=u_init,
                raw_disp=raw, raw_off=raw_off, disp=pset.displacement, off=pset.offset,
                mar=pset.mean_abs_residual, valid=pset.valid, hinv=pset.hessian_inv,
                mean_t=pset.template_mean, reset=was_reset, dense=flow)


def gen_search():
    cfg = synth.CONFIGS["c1"]
    f1, f2, gt = synth.make_pair(7, 109, 256, 12.0, True, 10.0)
    # level 1 (128x54) with a coarse init from the (scaled) ground truth
    coarse = np.ascontiguousarray(gt[::4, ::4][:27, :64] * 0.25)
    d = search_case(f1, f2, 1, 8, 0.5, 32, coarse)
    d.update({f"in_{k}": v for k, v in dict(f1=f1, f2=f2, coarse=coarse).items()})
    save("search_c1_like.npz", **d)
    # ps 12 / 0.75 / 128 iterations at full resolution of a small pair
    f1, f2, gt = synth.make_pair(8, 96, 160, 6.0, True, 6.0)
    coarse = gt[::2, ::2] * 0.5
    d = search_case(f1, f2, 0, 12, 0.75, 128, coarse)
    d.update({f"in_{k}": v for k, v in dict(f1=f1, f2=f2, coarse=coarse).items()})
    save("search_c2_like.npz", **d)
    # no init (coarsest scale), huber norm and l1 norm
    for norm in ("huber", "l1"):
        d = search_case(f1, f2, 0, 8, 0.3, 16, None, norm=norm)
        d.update({f"in_{k}": v for k, v in dict(f1=f1, f2=f2).items()})
        save(f"search_{norm}.npz", **d)


def gen_refine():
    f1, f2, gt = synth.make_pair(9, 48, 80, 4.0, True, 4.0)
    pyr1 = core.build_pyramid(f1, 0)
    pyr2 = core.build_pyramid(f2, 0)
    rng = np.random.default_rng(9)
    init = gt + rng.normal(0, 0.5, size=gt.shape)
    d = dict(f1=f1, f2=f2, init=init)
    d["refined_s0"] = variational.refine(init, pyr1[0], pyr2[0], core.VarParams(), 0)
    d["refined_s2"] = variational.refine(init, pyr1[0], pyr2[0], core.VarParams(), 2)
    d["refined_fixed1"] = variational.refine(init, pyr1[0], pyr2[0],
                                             VarParamsFixed(fixed_outer=1), 4)
    # the packed tensors and the assembled system at the init flow
    u = np.ascontiguousarray(init[:, :, 0])
    v = np.ascontiguousarray(init[:, :, 1])
    tens = variational._packed_tensors_uv(pyr1[0], pyr2[0], u, v,
                                          variational._second_derivatives(pyr1[0]),
                                          variational._second_derivatives(pyr2[0]))
    h, w = u.shape
    sysm = [np.empty((h, w)) for _ in range(6)]
    variational._assemble_system(tens, u, v, 5.0, 10.0, 10.0, 1e-3, *sysm)
    d["tens"] = tens
    d["sys"] = np.stack(sysm)
    du = np.zeros((h, w))
    dv = np.zeros((h, w))
    variational._sor_sweeps(u, v, du, dv, *sysm, 1.6, 5, False)
    d["sor_du"] = du
    d["sor_dv"] = dv
    save("refine.npz", **d)


def gen_e2e_small():
    """Small end-to-end pairs with each config's operating point."""
    cases = {
        # name: (cfg, h, w, coarsest, outer_fixed)
        "c0": ("c0", 112, 256, 3, 1),
        "c0_default_outer": ("c0", 112, 256, 3, None),
        "c1": ("c1", 109, 256, 3, 1),
        "c2": ("c2", 96, 160, 3, 1),
        "c3": ("c3", 135, 240, 4, 1),
        "c4": ("c4", 135, 240, 3, 1),
    }
    for name, (cn, h, w, coarsest, outer) in cases.items():
        cfg = synth.CONFIGS[cn]
        scale = w / cfg.width
        f1, f2, _ = synth.make_pair(11, h, w, max(2.0, cfg.maxmag * scale * 2), cfg.rects,
                                    max(2.0, cfg.rmax * scale * 2))
        params = ref_params(cfg, outer, coarsest)
        flow = pipeline.dis_flow(f1, f2, params)
        save(f"e2e_{name}.npz", f1=f1, f2=f2, flow=flow, patch_size=cfg.patch_size,
             overlap=cfg.overlap, iterations=cfg.iterations, finest=cfg.finest_scale,
             coarsest=coarsest, outer=-1 if outer is None else outer)


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def gen_full_hashes():
    """Full-size config pairs through the reference: sha256 of the flow
    bytes + summary statistics (the flows themselves are too large)."""
    rows = []
    plan = [("c0", 0, 1), ("c1", 0, 2), ("c2", 0, 1), ("c3", 0, 1), ("c4", 0, 1)]
    for cn, first, count in plan:
        cfg = synth.CONFIGS[cn]
        f1, f2 = synth.make_batch(cfg, seed=0, count=count, first=first)
        params = ref_params(cfg, 1)
        for i in range(count):
            flow = pipeline.dis_flow(f1[i], f2[i], params)
            rows.append((cn, first + i, digest(f1[i]), digest(f2[i]), digest(flow),
                         float(np.abs(flow).mean()), float(np.abs(flow).max())))
            print(rows[-1])
    save("full_hashes.npz", cfg=np.array([r[0] for r in rows]),
         pair=np.array([r[1] for r in rows]), f1_sha=np.array([r[2] for r in rows]),
         f2_sha=np.array([r[3] for r in rows]), flow_sha=np.array([r[4] for r in rows]),
         flow_absmean=np.array([r[5] for r in rows]), flow_absmax=np.array([r[6] for r in rows]))


def smooth_field(rng, h, w, mag, sigma=6.0):
    from scipy.ndimage import gaussian_filter

    f = np.stack([gaussian_filter(rng.standard_normal((h, w)), sigma) for _ in range(2)], -1)
    return f * (mag / max(1e-12, np.abs(f).max()))


def gen_compose():
    """compose_flows (pipeline.py:186-199) on smooth fields, fields that
    push samples outside the raster (clamping), and a 1-row field."""
    rng = np.random.default_rng(300)
    d = {}
    for k, (h, w, mag) in enumerate([(37, 53, 3.0), (29, 41, 40.0), (1, 17, 5.0)]):
        ab = smooth_field(rng, h, w, mag) if h > 1 else rng.uniform(-mag, mag, (h, w, 2))
        bc = smooth_field(rng, h, w, mag) if h > 1 else rng.uniform(-mag, mag, (h, w, 2))
        d[f"ab{k}"] = ab
        d[f"bc{k}"] = bc
        d[f"out{k}"] = pipeline.compose_flows(ab, bc)
    save("next_compose.npz", **d)


def _params_dict(p):
    vp = p.variational
    return dict(patch_size=p.patch_size, overlap=p.overlap, iterations=p.iterations,
                finest=p.finest_scale, coarsest=p.coarsest_scale,
                mean_norm=int(p.use_mean_normalization), norm=p.residual_norm,
                variational=int(vp is not None),
                outer=-1 if vp is None or not isinstance(vp, VarParamsFixed) else vp.fixed_outer,
                bidirectional=int(p.bidirectional), mode=p.mode)


def gen_stereo():
    """dis_stereo (pipeline.py:166-183) end to end, and the horizontal-only
    stages: conditioning (inverse_search.py:259-264) and SOR
    (variational.py:161)."""
    cases = [
        # (seed, h, w, maxdisp, params)
        (20, 96, 160, 6.0, dataclasses.replace(core.DisParams.preset(2, stereo=True),
                                               coarsest_scale=3)),
        (21, 109, 256, 10.0, core.DisParams(patch_size=12, overlap=0.75, iterations=32,
                                            finest_scale=0, coarsest_scale=3,
                                            variational=VarParamsFixed(fixed_outer=1),
                                            mode="stereo")),
        (22, 80, 128, 5.0, core.DisParams(patch_size=8, overlap=0.5, iterations=16,
                                          finest_scale=1, coarsest_scale=3, variational=None,
                                          mode="stereo")),
        # flow-mode params through dis_stereo (the reference does not check mode)
        (23, 96, 160, 6.0, core.DisParams(patch_size=8, overlap=0.5, iterations=16,
                                          finest_scale=1, coarsest_scale=3,
                                          variational=VarParamsFixed(fixed_outer=1))),
    ]
    for k, (seed, h, w, md, params) in enumerate(cases):
        f1, f2, _ = synth.make_stereo_pair(seed, h, w, md)
        flow = pipeline.dis_stereo(f1, f2, params)
        save(f"next_stereo_{k}.npz", f1=f1, f2=f2, flow=flow, **_params_dict(params))
    # horizontal SOR on the refine.npz system
    g = np.load(os.path.join(OUT, "refine.npz"))
    init = g["init"]
    u = np.ascontiguousarray(init[:, :, 0])
    v = np.ascontiguousarray(init[:, :, 1])
    sysm = [np.ascontiguousarray(x) for x in g["sys"]]
    du = np.zeros_like(u)
    dv = np.zeros_like(u)
    variational._sor_sweeps(u, v, du, dv, *sysm, 1.6, 5, True)
    f1, f2 = g["f1"], g["f2"]
    pyr1 = core.build_pyramid(f1, 0)
    pyr2 = core.build_pyramid(f2, 0)
    ref_h = variational.refine(init, pyr1[0], pyr2[0], VarParamsFixed(fixed_outer=2), 0,
                               horizontal_only=True)
    # horizontal conditioning on a textured level
    pset = inverse_search.precompute_patch_set(pyr1[0], np.arange(0, 70, 5.0),
                                               np.arange(0, 70, 5.0) * 0.5, 8,
                                               horizontal_only=True)
    save("next_stereo_stages.npz", sor_du=du, sor_dv=dv, refined_h=ref_h,
         cond_valid=pset.valid, cond_hinv=pset.hessian_inv, cond_hess=pset.hessian)


def gen_bidir():
    """bidirectional densification: densify_bidirectional
    (densification.py:194-234) on explicit patch sets, and dis_flow with
    bidirectional=True end to end."""
    rng = np.random.default_rng(400)
    f1, f2, gt = synth.make_pair(24, 54, 128, 6.0, True, 6.0)
    pyr1 = core.build_pyramid(f1, 0)
    pyr2 = core.build_pyramid(f2, 0)
    d = dict(f1=f1, f2=f2)
    for k, (ps, ov, mag) in enumerate([(8, 0.5, 3.0), (12, 0.75, 9.0), (8, 0.3, 40.0)]):
        fg = densification.create_grid(128, 54, ps, ov)
        n = fg.starts.shape[0]
        fdisp = rng.normal(0, mag, (n, 2))
        fdisp[::7] = np.round(fdisp[::7])  # integer displacements: closed windows
        bdisp = rng.normal(0, mag, (n, 2))
        bdisp[::5] = np.round(bdisp[::5])
        foff = rng.normal(0, 2, n)
        boff = rng.normal(0, 2, n)
        d[f"ps{k}"] = ps
        d[f"ov{k}"] = ov
        d[f"fdisp{k}"] = fdisp
        d[f"bdisp{k}"] = bdisp
        d[f"foff{k}"] = foff
        d[f"boff{k}"] = boff
        d[f"flow{k}"] = densification.densify_bidirectional(
            fg, fdisp, foff, fg, bdisp, boff, pyr1[0].image, pyr2[0].image)
    save("next_bidir_stage.npz", **d)
    cases = [
        (25, 109, 256, 8.0, core.DisParams(patch_size=8, overlap=0.5, iterations=32,
                                           finest_scale=1, coarsest_scale=3,
                                           variational=VarParamsFixed(fixed_outer=1),
                                           bidirectional=True)),
        (26, 96, 160, 6.0, core.DisParams(patch_size=12, overlap=0.75, iterations=64,
                                          finest_scale=0, coarsest_scale=3,
                                          variational=VarParamsFixed(fixed_outer=1),
                                          bidirectional=True)),
        (27, 80, 128, 5.0, core.DisParams(patch_size=8, overlap=0.3, iterations=16,
                                          finest_scale=2, coarsest_scale=3, variational=None,
                                          bidirectional=True)),
        (28, 96, 160, 6.0, dataclasses.replace(core.DisParams.preset(2), coarsest_scale=3,
                                               bidirectional=True)),
    ]
    for k, (seed, h, w, mag, params) in enumerate(cases):
        f1, f2, _ = synth.make_pair(seed, h, w, mag, True, mag)
        flow = pipeline.dis_flow(f1, f2, params)
        save(f"next_bidir_{k}.npz", f1=f1, f2=f2, flow=flow, **_params_dict(params))


def gen_sparse():
    """sparse_correspondences (pipeline.py:230-287): densified and per-seed
    chain modes; seeds inside, on the border, fractional and outside."""
    f1, f2, _ = synth.make_pair(29, 109, 256, 8.0, True, 8.0)
    rng = np.random.default_rng(500)
    seeds = np.concatenate([
        rng.uniform([0, 0], [255, 108], (40, 2)),
        np.array([[0.0, 0.0], [255.0, 108.0], [255.0, 0.0], [0.0, 108.0], [3.5, 100.25],
                  [-0.5, 10.0], [256.0, 5.0], [10.0, -1e-9], [10.0, 108.5]]),
    ])
    cases = {
        "dense": core.DisParams(patch_size=8, overlap=0.5, iterations=32, finest_scale=1,
                                coarsest_scale=3, variational=VarParamsFixed(fixed_outer=1)),
        "chain": core.DisParams(patch_size=8, overlap=0.5, iterations=32, finest_scale=1,
                                coarsest_scale=3, use_densification=False),
        "chain_s0": core.DisParams(patch_size=12, overlap=0.75, iterations=64, finest_scale=0,
                                   coarsest_scale=3, use_densification=False),
        "dense_bidir": core.DisParams(patch_size=8, overlap=0.3, iterations=16,
                                      finest_scale=2, coarsest_scale=3, variational=None,
                                      bidirectional=True),
    }
    d = dict(f1=f1, f2=f2, seeds=seeds)
    for name, p in cases.items():
        m = pipeline.sparse_correspondences(f1, f2, seeds, p)
        d[f"{name}_disp"] = np.array([mm.displacement for mm in m])
        d[f"{name}_valid"] = np.array([mm.valid for mm in m])
        d[f"{name}_seed"] = np.array([mm.seed for mm in m])
        for k, v in _params_dict(p).items():
            d[f"{name}_{k}"] = v
        d[f"{name}_dens"] = int(p.use_densification)
    save("next_sparse.npz", **d)


def gen_downscale():
    """downscale > 2 (core.py:88-128 box means over k x k blocks, init_patches
    densification.py:82-95, upsample_flow core.py:178-190, the sparse chain
    pipeline.py:202-231): pyramids for k = 3, 4, 8, 9 and end-to-end flows,
    stereo and sparse correspondences for k = 3 and 4."""
    rng = np.random.default_rng(700)
    d = {}
    for k, (h, w) in {3: (97, 131), 4: (131, 257), 8: (130, 140), 9: (200, 190)}.items():
        img = rng.uniform(0, 255, (h, w))
        pyr = core.build_pyramid(img, 2 if k < 8 else 1, downscale=k)
        d[f"pyr{k}_img"] = img
        for s in range(len(pyr.levels)):
            d[f"pyr{k}_L{s}"] = pyr[s].image
            d[f"pyr{k}_L{s}_gx"] = pyr[s].grad_x
            d[f"pyr{k}_L{s}_gy"] = pyr[s].grad_y
    cases = {
        # name: (seed, h, w, maxmag, params)
        "f3": (40, 109, 256, 6.0, core.DisParams(
            patch_size=8, overlap=0.5, iterations=32, finest_scale=1, coarsest_scale=2,
            downscale=3, variational=VarParamsFixed(fixed_outer=1))),
        "f3_default_outer": (41, 120, 200, 5.0, core.DisParams(
            patch_size=8, overlap=0.3, iterations=16, finest_scale=1, coarsest_scale=2,
            downscale=3)),
        "f4": (42, 160, 300, 8.0, core.DisParams(
            patch_size=8, overlap=0.5, iterations=32, finest_scale=1, coarsest_scale=2,
            downscale=4, variational=VarParamsFixed(fixed_outer=1))),
        "f3_s0": (43, 120, 200, 5.0, core.DisParams(
            patch_size=12, overlap=0.75, iterations=64, finest_scale=0, coarsest_scale=2,
            downscale=3, variational=VarParamsFixed(fixed_outer=1))),
        "f3_bidir": (44, 109, 256, 6.0, core.DisParams(
            patch_size=8, overlap=0.5, iterations=16, finest_scale=1, coarsest_scale=2,
            downscale=3, variational=VarParamsFixed(fixed_outer=1), bidirectional=True)),
    }
    for name, (seed, h, w, mm, p) in cases.items():
        f1, f2, _ = synth.make_pair(seed, h, w, mm, True, mm)
        d[f"{name}_f1"] = f1
        d[f"{name}_f2"] = f2
        d[f"{name}_flow"] = pipeline.dis_flow(f1, f2, p)
        for kk, v in _params_dict(p).items():
            d[f"{name}_{kk}"] = v
        d[f"{name}_downscale"] = p.downscale
    f1, f2, _ = synth.make_stereo_pair(45, 96, 200, 6.0)
    sp = core.DisParams(patch_size=8, overlap=0.5, iterations=16, finest_scale=1,
                        coarsest_scale=2, downscale=3, mode="stereo",
                        variational=VarParamsFixed(fixed_outer=1))
    d["st3_f1"], d["st3_f2"] = f1, f2
    d["st3_flow"] = pipeline.dis_stereo(f1, f2, sp)
    f1, f2, _ = synth.make_pair(46, 109, 256, 6.0, True, 6.0)
    seeds = np.concatenate([rng.uniform([0, 0], [255, 108], (30, 2)),
                            np.array([[0.0, 0.0], [255.0, 108.0], [-1.0, 3.0]])])
    d["sp_f1"], d["sp_f2"], d["sp_seeds"] = f1, f2, seeds
    for name, dens in (("sp_dense", True), ("sp_chain", False)):
        p = core.DisParams(patch_size=8, overlap=0.5, iterations=32, finest_scale=1,
                           coarsest_scale=2, downscale=3, use_densification=dens,
                           variational=VarParamsFixed(fixed_outer=1))
        m = pipeline.sparse_correspondences(f1, f2, seeds, p)
        d[f"{name}_disp"] = np.array([mm.displacement for mm in m])
        d[f"{name}_valid"] = np.array([mm.valid for mm in m])
    save("downscale.npz", **d)


def gen_stage_search():
    """The inverse-search stage functions (inverse_search.py:306-494) at real
    (non-grid) window origins, all three residual norms, with and without
    mean normalisation, plus refresh_patch_stats on a selection and the
    single-patch interface."""
    f1, f2, _ = synth.make_pair(50, 96, 160, 4.0, True, 4.0)
    lv1 = core.build_pyramid(f1, 0)[0]
    lv2 = core.build_pyramid(f2, 0)[0]
    rng = np.random.default_rng(51)
    n = 300
    xs = rng.uniform(-3.0, 160.0 - 6.0, n)
    ys = rng.uniform(-3.0, 96.0 - 6.0, n)
    xs[:10] = np.floor(xs[:10])  # some integer origins too
    d = dict(f1=f1, f2=f2, xs=xs, ys=ys)
    for ps in (8, 12):
        for hz in (False, True):
            pset = inverse_search.precompute_patch_set(lv1, xs, ys, ps, horizontal_only=hz)
            tag = f"ps{ps}_{'h' if hz else 'f'}"
            d[f"{tag}_tmpl"] = pset.templates
            d[f"{tag}_sdx"] = pset.steep_x
            d[f"{tag}_sdy"] = pset.steep_y
            d[f"{tag}_hess"] = pset.hessian
            d[f"{tag}_hinv"] = pset.hessian_inv
            d[f"{tag}_mean"] = pset.template_mean
            d[f"{tag}_valid"] = pset.valid
    init = rng.normal(0, 1.5, (n, 2))
    d["init"] = init
    for norm in ("l2", "l1", "huber"):
        for mn in (True, False):
            pset = inverse_search.precompute_patch_set(lv1, xs, ys, 8)
            pset.init_displacement = init.copy()
            inverse_search.optimize_patch_set(pset, lv2, 24, residual_norm=norm, huber_b=2.0,
                                              mean_normalization=mn)
            tag = f"opt_{norm}_{int(mn)}"
            d[f"{tag}_disp"] = pset.displacement.copy()
            d[f"{tag}_off"] = pset.offset.copy()
            d[f"{tag}_mar"] = pset.mean_abs_residual.copy()
            if norm == "l2" and mn:
                sel = rng.uniform(0, 1, n) < 0.3
                kept = densification.reset_outliers(pset.displacement, init, 8)
                pset.displacement = kept
                inverse_search.refresh_patch_stats(pset, lv2, sel, True)
                d["refresh_sel"] = sel
                d["refresh_disp"] = kept
                d["refresh_off"] = pset.offset.copy()
                d["refresh_mar"] = pset.mean_abs_residual.copy()
    st = inverse_search.precompute_patch(lv1, (70.3, 40.8), 8)
    st = dataclasses.replace(st, init_displacement=np.array([1.25, -0.5]))
    out = inverse_search.optimize_patch(st, lv2, 32, residual_norm="huber", huber_b=1.5)
    d["single_tmpl"] = st.template
    d["single_sd"] = st.steepest_descent
    d["single_hinv"] = st.hessian_inverse
    d["single_disp"] = out.displacement
    d["single_off"] = np.array(out.mean_offset)
    d["single_mar"] = np.array(out.mean_abs_residual)
    save("stage_search.npz", **d)


def gen_flowio():
    """flowio.py: .flo bytes written by the reference, images decoded by it
    (P5 8/16-bit with header comments, P6 luminance), written PGM/PPM bytes."""
    import tempfile

    from disflow import flowio

    rng = np.random.default_rng(600)
    d = {}
    flow = rng.normal(0, 5, (7, 11, 2))
    flow[2, 3] = [1e10, 1e10]  # sentinel passes through
    with tempfile.TemporaryDirectory() as td:
        fp = os.path.join(td, "a.flo")
        flowio.write_flo(flow, fp)
        d["flo_in"] = flow
        d["flo_bytes"] = np.frombuffer(open(fp, "rb").read(), dtype=np.uint8)
        d["flo_read"] = flowio.read_flo(fp)
        pgm8 = rng.integers(0, 256, (9, 13), dtype=np.uint8)
        raw = b"P5\n# a comment\n13 9\n# another\n255\n" + pgm8.tobytes()
        d["pgm8_bytes"] = np.frombuffer(raw, dtype=np.uint8)
        open(os.path.join(td, "a.pgm"), "wb").write(raw)
        d["pgm8_img"] = flowio.read_image(os.path.join(td, "a.pgm"))
        pgm16 = rng.integers(0, 1000, (5, 6)).astype(">u2")
        raw = b"P5 6 5 999\n" + pgm16.tobytes()
        d["pgm16_bytes"] = np.frombuffer(raw, dtype=np.uint8)
        open(os.path.join(td, "b.pgm"), "wb").write(raw)
        d["pgm16_img"] = flowio.read_image(os.path.join(td, "b.pgm"))
        ppm = rng.integers(0, 256, (4, 5, 3), dtype=np.uint8)
        raw = b"P6\n5 4\n255\n" + ppm.tobytes()
        d["ppm_bytes"] = np.frombuffer(raw, dtype=np.uint8)
        open(os.path.join(td, "c.ppm"), "wb").write(raw)
        d["ppm_img"] = flowio.read_image(os.path.join(td, "c.ppm"))
        img = rng.uniform(-20, 280, (6, 8))
        flowio.write_image(img, os.path.join(td, "d.pgm"))
        d["wimg_in"] = img
        d["wimg_bytes"] = np.frombuffer(open(os.path.join(td, "d.pgm"), "rb").read(), np.uint8)
        rgb = rng.uniform(0, 255, (3, 4, 3))
        flowio.write_image(rgb, os.path.join(td, "e.ppm"))
        d["wrgb_in"] = rgb
        d["wrgb_bytes"] = np.frombuffer(open(os.path.join(td, "e.ppm"), "rb").read(), np.uint8)
        d["mask"] = flowio.flow_valid_mask(flow)
    save("next_flowio.npz", **d)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    which = sys.argv[1:] or ["pyramid", "samplers", "search", "refine", "e2e", "full",
                             "compose", "stereo", "bidir", "sparse", "flowio", "downscale",
                             "stage_search"]
    pipeline.warmup()
    if "pyramid" in which:
        gen_pyramid()
    if "samplers" in which:
        gen_samplers()
    if "search" in which:
        gen_search()
    if "refine" in which:
        gen_refine()
    if "e2e" in which:
        gen_e2e_small()
    if "full" in which:
        gen_full_hashes()
    if "compose" in which:
        gen_compose()
    if "stereo" in which:
        gen_stereo()
    if "bidir" in which:
        gen_bidir()
    if "sparse" in which:
        gen_sparse()
    if "flowio" in which:
        gen_flowio()
    if "downscale" in which:
        gen_downscale()
    if "stage_search" in which:
        gen_stage_search()
