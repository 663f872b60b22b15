"""CUDA path vs the oracle / reference goldens — bit-exact (float64 in the
reference's operation order; the tolerance for every comparison here is
zero: np.array_equal).  All calls go through the C ABI (libdis_b200.so)."""

import dataclasses
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


@pytest.fixture(scope="module")
def st(torch):
    from paper_1603_03590_b200 import stages

    return stages


def _np(t):
    return t.detach().cpu().numpy()


def test_exact_div_matches_ieee(torch):
    """The SOR/densify/patch-search division helper is bit-identical to IEEE
    division over ~50M operand pairs: SOR-like magnitudes, random exponents
    over the whole fast-path range, tiny/huge/zero numerators (fallback)."""
    from paper_1603_03590_b200 import _lib

    rng = np.random.default_rng(123)
    parts = []
    for _ in range(6):
        n = 8_000_000
        num = rng.standard_normal(n) * 10.0 ** rng.uniform(-12, 8, n)
        den = 10.0 ** rng.uniform(-11.9, 10, n) * rng.uniform(1, 2, n)
        parts.append((num, den))
    e1 = np.ldexp(rng.uniform(1, 2, 2_000_000), rng.integers(-1000, 1000, 2_000_000))
    e2 = np.ldexp(rng.uniform(1, 2, 2_000_000), rng.integers(-1000, 1000, 2_000_000))
    parts.append((e1 * np.sign(rng.standard_normal(2_000_000)), e2))
    special = np.array([0.0, -0.0, 1e-300, -1e-300, 5e-324, 1e300, 1.0, -1.0, 3.0, np.nextafter(1, 2)])
    parts.append((np.repeat(special, len(special)), np.tile(np.abs(special[special != 0][:8]).tolist() + [2.0, 7.0], len(special))))
    L = _lib.lib()
    for num, den in parts:
        n_t = torch.tensor(num, device="cuda")
        d_t = torch.tensor(den, device="cuda")
        fast = torch.empty_like(n_t)
        ieee = torch.empty_like(n_t)
        _lib.check(L.dis_selftest_div(n_t.data_ptr(), d_t.data_ptr(), fast.data_ptr(),
                                      ieee.data_ptr(), n_t.numel(), None))
        f = fast.cpu().numpy().view(np.uint64)
        i = ieee.cpu().numpy().view(np.uint64)
        bad = np.flatnonzero(f != i)
        assert bad.size == 0, (num[bad[:5]], den[bad[:5]])


def test_pyramid_bit_exact(torch, st):
    g = golden("pyramid.npz")
    levels = st.build_pyramid(g["img"][None], 4, finest=0)
    for s, lv in enumerate(levels):
        assert np.array_equal(_np(lv["img"])[0], g[f"L{s}_img"]), s
        assert np.array_equal(_np(lv["gx"])[0], g[f"L{s}_gx"]), s
        assert np.array_equal(_np(lv["gy"])[0], g[f"L{s}_gy"]), s
        assert np.array_equal(_np(lv["dd"])[0], g[f"L{s}_dd"]), s


def test_pyramid_level1_from_frames_and_f64_u8_inputs(torch, st, orc):
    rng = np.random.default_rng(5)
    for dt in (np.float32, np.float64, np.uint8):
        img = (rng.uniform(0, 255, size=(2, 67, 95))).astype(dt)
        lv = st.build_pyramid(img, 3, finest=1)
        for b in range(2):
            ref = orc.build_pyramid(img[b].astype(np.float64), 3)
            for s in range(1, 4):
                assert np.array_equal(_np(lv[s]["img"])[b], ref[s][0])
                assert np.array_equal(_np(lv[s]["gx"])[b], ref[s][1])
                assert np.array_equal(_np(lv[s]["gy"])[b], ref[s][2])


def test_box_mean_order(torch, st):
    g = golden("pyramid.npz")
    big = np.random.default_rng(1000).uniform(0, 255, size=(200, 400))
    lv = st.build_pyramid(big[None], 1, finest=2)
    assert np.array_equal(_np(lv[1]["img"])[0], g["box_out"])


def test_nonfinite_input_raises(torch, st):
    img = np.zeros((1, 16, 16), dtype=np.float32)
    img[0, 3, 4] = np.nan
    with pytest.raises(ValueError):
        st.build_pyramid(img, 1)


@pytest.mark.parametrize("h,w", [(17, 23), (16, 23), (17, 24), (9, 2047)])
def test_nonfinite_input_found_at_every_position(torch, st, h, w):
    # the level-1 pass reads the frames two output pixels at a time and checks
    # the odd last column / row separately: a non-finite value anywhere raises
    rng = np.random.default_rng(h * w)
    spots = [(0, 0), (h - 1, w - 1), (h - 1, 0), (0, w - 1), (h // 2, w // 2)]
    spots += [(int(rng.integers(h)), int(rng.integers(w))) for _ in range(3)]
    for dtype in (np.float32, np.float64):
        for y, x in spots:
            img = rng.uniform(0, 255, (2, h, w)).astype(dtype)
            img[1, y, x] = np.inf
            with pytest.raises(ValueError):
                st.build_pyramid(img, 1)
        st.build_pyramid(rng.uniform(0, 255, (2, h, w)).astype(dtype), 1)  # finite: fine


def test_upsample_bit_exact(torch, st):
    g = golden("samplers.npz")
    f = torch.tensor(g["flow"], device="cuda")
    u, v = f[..., 0][None].contiguous(), f[..., 1][None].contiguous()
    for key, (hn, wn) in (("up_27x35", (27, 35)), ("up_26x34", (26, 34))):
        ou, ov = st.upsample_flow(u, v, wn, hn)
        assert np.array_equal(np.stack([_np(ou)[0], _np(ov)[0]], -1), g[key])


def test_grid_axis_matches_reference(torch, st):
    g = golden("samplers.npz")
    off = 0
    for dim, ps, ov, cnt in zip(g["grid_dims"], g["grid_ps"], g["grid_ov"], g["grid_counts"]):
        o = st.grid_axis(int(dim), int(ps), float(ov))
        assert np.array_equal(o, g["grid_origins"][off:off + cnt])
        off += cnt


@pytest.mark.parametrize("name,s,ps,ov,iters,norm", [
    ("search_c1_like.npz", 1, 8, 0.5, 32, "l2"),
    ("search_c2_like.npz", 0, 12, 0.75, 128, "l2"),
    ("search_huber.npz", 0, 8, 0.3, 16, "huber"),
    ("search_l1.npz", 0, 8, 0.3, 16, "l1"),
])
def test_patch_search_and_densify_bit_exact(torch, st, name, s, ps, ov, iters, norm):
    g = golden(name)
    params = DisParams(patch_size=ps, overlap=ov, iterations=iters, finest_scale=0,
                       coarsest_scale=max(s, 1), residual_norm=norm, huber_b=1.0)
    l1 = st.build_pyramid(g["in_f1"][None], s, finest=s)[s]
    l2 = st.build_pyramid(g["in_f2"][None], s, finest=s)[s]
    cu = cv = None
    if "in_coarse" in g.files:
        c = torch.tensor(g["in_coarse"], device="cuda")
        cu, cv = c[..., 0][None].contiguous(), c[..., 1][None].contiguous()
    r = st.patch_search(l1, l2["img"], params, cu, cv)
    assert np.array_equal(r["x_origins"], g["x_origins"])
    assert np.array_equal(r["y_origins"], g["y_origins"])
    init = np.stack([_np(r["init_u"])[0], _np(r["init_v"])[0]], -1)
    assert np.array_equal(init, g["init"])
    assert np.array_equal(_np(r["valid"])[0].astype(bool), g["valid"])
    disp = np.stack([_np(r["u"])[0], _np(r["v"])[0]], -1)
    assert np.array_equal(disp, g["disp"])
    assert np.array_equal(_np(r["off"])[0], g["off"])
    assert np.array_equal(_np(r["mar"])[0], g["mar"])
    fu, fv = st.densify(l1["img"], l2["img"], params, r["u"], r["v"], r["off"])
    assert np.array_equal(np.stack([_np(fu)[0], _np(fv)[0]], -1), g["dense"])


def test_refine_bit_exact(torch, st):
    g = golden("refine.npz")
    l1 = st.build_pyramid(g["f1"][None], 0)[0]
    l2 = st.build_pyramid(g["f2"][None], 0)[0]
    init = torch.tensor(g["init"], device="cuda")
    u0, v0 = init[..., 0][None].contiguous(), init[..., 1][None].contiguous()
    p = DisParams(variational=VarParams())
    for key, outer in (("refined_s0", 1), ("refined_s2", 3), ("refined_fixed1", 1)):
        u, v = st.refine(u0, v0, l1, l2, p, outer)
        assert np.array_equal(np.stack([_np(u)[0], _np(v)[0]], -1), g[key]), key


@pytest.mark.parametrize("sweeps", [1, 3, 8, 11])
def test_refine_sweep_counts_vs_oracle(torch, st, orc, sweeps):
    g = golden("refine.npz")
    l1 = st.build_pyramid(g["f1"][None], 0)[0]
    l2 = st.build_pyramid(g["f2"][None], 0)[0]
    init = torch.tensor(g["init"], device="cuda")
    u0, v0 = init[..., 0][None].contiguous(), init[..., 1][None].contiguous()
    vp = VarParams(inner_sor_iters=sweeps)
    u, v = st.refine(u0, v0, l1, l2, DisParams(variational=vp), 2)
    lv1 = orc.build_pyramid(g["f1"], 0)[0]
    lv2 = orc.build_pyramid(g["f2"], 0)[0]
    want = orc.refine(g["init"], lv1, lv2, vp, 2)
    assert np.array_equal(np.stack([_np(u)[0], _np(v)[0]], -1), want)


def _params_from(g):
    outer = int(g["outer"])
    return DisParams(
        patch_size=int(g["patch_size"]), overlap=float(g["overlap"]),
        iterations=int(g["iterations"]), finest_scale=int(g["finest"]),
        coarsest_scale=int(g["coarsest"]),
        variational=VarParams(outer_iters_fixed=None if outer < 0 else outer))


@pytest.mark.parametrize("case", ["c0", "c0_default_outer", "c1", "c2", "c3", "c4"])
def test_end_to_end_small_goldens(torch, case):
    from paper_1603_03590_b200 import dis_flow

    g = golden(f"e2e_{case}.npz")
    flow = dis_flow(g["f1"], g["f2"], _params_from(g))
    assert flow.dtype == np.float64
    assert np.array_equal(flow, g["flow"])


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.mark.parametrize("cfg_name", ["c0", "c1", "c2", "c3"])
def test_full_size_configs_match_reference_hashes(torch, cfg_name):
    """BASELINE configs at full size: the CUDA flow's sha256 equals the sha256
    of the reference's own output on the same pair (tests/golden)."""
    from paper_1603_03590_b200 import dis_flow_batch

    g = golden("full_hashes.npz")
    rows = [i for i, c in enumerate(g["cfg"]) if str(c) == cfg_name]
    cfg = synth.CONFIGS[cfg_name]
    first = min(int(g["pair"][i]) for i in rows)
    count = max(int(g["pair"][i]) for i in rows) - first + 1
    f1, f2 = synth.make_batch(cfg, seed=0, count=count, first=first)
    flow = dis_flow_batch(f1, f2, synth.dis_params(cfg)).cpu().numpy()
    for i in rows:
        k = int(g["pair"][i]) - first
        assert _sha(flow[k]) == str(g["flow_sha"][i]), (cfg_name, k)


@pytest.mark.parametrize("cfg_name,count", [("c1", 6), ("c2", 2), ("c3", 2)])
def test_batched_full_size_vs_oracle(torch, orc, cfg_name, count):
    """Several pairs in one batch (pair i uses seed i) against the oracle,
    bit-exact; checks batching does not couple pairs."""
    from paper_1603_03590_b200 import dis_flow_batch

    cfg = synth.CONFIGS[cfg_name]
    f1, f2 = synth.make_batch(cfg, seed=3, count=count)
    params = synth.dis_params(cfg)
    flow = dis_flow_batch(f1, f2, params).cpu().numpy()
    want = orc.dis_flow_batch_f32(f1, f2, params)
    for k in range(count):
        assert np.array_equal(flow[k], want[k]), (cfg_name, k)


def test_determinism_repeat_runs(torch):
    from paper_1603_03590_b200 import dis_flow_batch

    cfg = synth.CONFIGS["c1"]
    f1, f2 = synth.make_batch(cfg, seed=9, count=3, h=218, w=512)
    params = synth.dis_params(cfg, coarsest=4)
    a = dis_flow_batch(f1, f2, params).cpu().numpy()
    b = dis_flow_batch(f1, f2, params).cpu().numpy()
    assert np.array_equal(a, b)


def test_host_buffer_path_matches_device_path(torch):
    from paper_1603_03590_b200 import FlowEngine

    cfg = synth.CONFIGS["c0"]
    f1, f2 = synth.make_batch(cfg, seed=4, count=2)
    eng = FlowEngine(2, cfg.height, cfg.width, synth.dis_params(cfg))
    dev = eng.run(torch.from_numpy(f1).cuda(), torch.from_numpy(f2).cuda()).cpu().numpy()
    host = eng.run_host(f1, f2)
    assert np.array_equal(dev, host)


def test_host_path_graph_replay_with_pinned_buffers(torch):
    # repeated calls with the same pinned buffers are captured (second call)
    # and replayed (third on) as one CUDA graph inside the library
    from paper_1603_03590_b200 import FlowEngine

    cfg = synth.CONFIGS["c0"]
    f1, f2 = synth.make_batch(cfg, seed=7, count=3)
    eng = FlowEngine(3, cfg.height, cfg.width, synth.dis_params(cfg))
    want = eng.run(torch.from_numpy(f1).cuda(), torch.from_numpy(f2).cuda()).cpu().numpy()
    p1 = torch.from_numpy(f1).pin_memory()
    p2 = torch.from_numpy(f2).pin_memory()
    po = torch.empty((3, cfg.height, cfg.width, 2), dtype=torch.float64).pin_memory()
    for _ in range(4):
        po.zero_()
        eng.run_host(p1.numpy(), p2.numpy(), out=po.numpy())
        assert np.array_equal(po.numpy(), want)
    # new frame contents in the same buffers are picked up by the replay
    p1.copy_(p2)
    eng.run_host(p1.numpy(), p2.numpy(), out=po.numpy())
    same = eng.run(torch.from_numpy(f2).cuda(), torch.from_numpy(f2).cuda()).cpu().numpy()
    assert np.array_equal(po.numpy(), same)
    p1[0, 3, 3] = float("inf")
    with pytest.raises(ValueError):
        eng.run_host(p1.numpy(), p2.numpy(), out=po.numpy())


def test_graph_replay_matches_eager_and_reports_errors(torch):
    from paper_1603_03590_b200 import FlowEngine

    cfg = synth.CONFIGS["c0"]
    f1, f2 = synth.make_batch(cfg, seed=6, count=2)
    eng = FlowEngine(2, cfg.height, cfg.width, synth.dis_params(cfg))
    a, b = torch.from_numpy(f1).cuda(), torch.from_numpy(f2).cuda()
    eager = eng.run(a, b).cpu().numpy()
    out = torch.zeros((2, cfg.height, cfg.width, 2), dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(3):  # capture once, replay
        out.zero_()
        eng.run(a, b, out=out, stream=s, graph=True)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), eager)
    # new contents in the captured buffers: the replay recomputes them
    a.copy_(b)
    eng.run(a, b, out=out, stream=s, graph=True)
    assert np.array_equal(out.cpu().numpy(), eng.run(b, b).cpu().numpy())
    # the status word is reset and checked inside every replay
    a[0, 5, 5] = float("inf")
    with pytest.raises(ValueError):
        eng.run(a, b, out=out, stream=s, graph=True)


def test_error_types(torch):
    from paper_1603_03590_b200 import ParameterError, dis_flow

    a = np.zeros((64, 64), dtype=np.float32)
    with pytest.raises(ValueError):
        dis_flow(a, np.zeros((64, 65), dtype=np.float32))
    with pytest.raises(ParameterError):
        dis_flow(a, a, DisParams(patch_size=1))
    with pytest.raises(ValueError):  # coarsest level cannot hold the patch
        dis_flow(a, a, DisParams(coarsest_scale=5, finest_scale=3))
    bad = a.copy()
    bad[3, 3] = np.inf
    with pytest.raises(ValueError):
        dis_flow(bad, a, DisParams(coarsest_scale=2, finest_scale=1))


def test_mixed_dtype_pair_promotes_to_float64(torch, orc):
    """as_image converts both frames to float64 (core.py:65-72): a uint8
    frame1 with a float64 frame2 (fractional values) gives the oracle's flow
    on the float64 pair — frame2 is never narrowed to frame1's dtype."""
    from paper_1603_03590_b200 import FlowEngine, dis_flow

    cfg = synth.CONFIGS["c0"]
    f1, f2 = synth.make_batch(cfg, seed=21, count=1, h=109, w=256)
    a = np.clip(np.rint(f1[0]), 0, 255).astype(np.uint8)
    b = f2[0].astype(np.float64) + 0.25
    params = synth.dis_params(cfg, coarsest=3)
    params = dataclasses.replace(params, finest_scale=1)
    want = orc.dis_flow(a.astype(np.float64), b, params)
    assert np.array_equal(dis_flow(a, b, params), want)
    got_t = dis_flow(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), params)
    assert np.array_equal(got_t.cpu().numpy(), want)
    eng = FlowEngine(1, 109, 256, params)
    assert np.array_equal(eng.run_host(a[None], b[None])[0], want)
    # a NaN in the float64 frame2 is caught even though frame1 is uint8
    bad = b.copy()
    bad[7, 9] = np.nan
    with pytest.raises(ValueError):
        dis_flow(a, bad, params)


def test_engine_rejects_mismatched_buffers(torch):
    from paper_1603_03590_b200 import FlowEngine

    cfg = synth.CONFIGS["c1"]
    eng = FlowEngine(2, 64, 96, synth.dis_params(cfg, coarsest=2))
    f = np.zeros((2, 64, 96), dtype=np.float32)
    with pytest.raises(ValueError):
        eng.run_host(f[:1], f[:1])
    with pytest.raises(ValueError):
        eng.run_host(f, f, out=np.empty((2, 64, 96, 2), dtype=np.float16))  # (float32: opt-in)
    with pytest.raises(ValueError):
        eng.run_host(f, f, out=np.empty((2, 64, 96, 2), dtype=np.int64))
    with pytest.raises(ValueError):
        eng.run_host(f, f, out=np.empty((1, 64, 96, 2)))
    d = torch.zeros((2, 64, 96), device="cuda")
    with pytest.raises(ValueError):
        eng.run(d, d, out=torch.empty((2, 64, 96, 2), dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        eng.run(d, d, out=torch.empty((2, 96, 64, 2), dtype=torch.float64,
                                      device="cuda").transpose(1, 2))
    with pytest.raises(ValueError):
        eng.run(d, d, out=torch.empty((2, 64, 96, 2), dtype=torch.float64))  # host tensor


def test_default_stream_is_torch_current_stream(torch):
    """With no explicit stream the engine launches on torch's current stream,
    so work queued there before the call (the frames' producer) is ordered
    before the kernels."""
    from paper_1603_03590_b200 import FlowEngine

    cfg = synth.CONFIGS["c0"]
    f1, f2 = synth.make_batch(cfg, seed=8, count=1)
    eng = FlowEngine(1, cfg.height, cfg.width, synth.dis_params(cfg))
    want = eng.run(torch.from_numpy(f1).cuda(), torch.from_numpy(f2).cuda()).cpu().numpy()
    s = torch.cuda.Stream()
    h1 = torch.from_numpy(f1).pin_memory()
    with torch.cuda.stream(s):
        a = torch.empty_like(h1, device="cuda")
        torch.cuda._sleep(50_000_000)  # keep the side stream busy before the copy
        a.copy_(h1, non_blocking=True)
        b = torch.from_numpy(f2).cuda()
        got = eng.run(a, b)
        res = got.cpu().numpy()
    assert np.array_equal(res, want)


@pytest.mark.parametrize("h,w,coarsest,finest", [(67, 95, 3, 1), (436, 1024, 5, 1), (64, 130, 4, 0),
                                                 (256, 2049, 7, 1), (1080, 1920, 7, 2)])
def test_fused_pyramid_matches_oracle(torch, st, orc, h, w, coarsest, finest):
    """The flow path's fused pyramid (one tile kernel for the base level, its
    gradients and the coarser images from shared memory, one launch for the
    coarser gradients; deeper levels by box-mean launches): every level's
    image and gradients bit-exact against the oracle, odd sizes, f32/f64/u8
    frames, base level 0 and 1, pyramids deeper than one tile's halvings."""
    rng = np.random.default_rng(h + w)
    for dt in (np.float32, np.float64, np.uint8):
        img = rng.uniform(0, 255, size=(2, h, w)).astype(dt)
        lv = st.build_pyramid(img, coarsest, finest=finest, second_derivatives=False,
                              level0=finest == 0)
        for b in range(2):
            ref = orc.build_pyramid(img[b].astype(np.float64), coarsest)
            for s in range(0 if finest == 0 else 1, coarsest + 1):
                assert np.array_equal(_np(lv[s]["img"])[b], ref[s][0]), (dt, b, s)
                if s >= finest:
                    assert np.array_equal(_np(lv[s]["gx"])[b], ref[s][1]), (dt, b, s)
                    assert np.array_equal(_np(lv[s]["gy"])[b], ref[s][2]), (dt, b, s)


@pytest.mark.parametrize("h,w", [(67, 95), (436, 1024), (65, 130)])
def test_fused_pyramid_nonfinite_anywhere(torch, st, h, w):
    rng = np.random.default_rng(h * 7 + w)
    spots = [(0, 0), (h - 1, w - 1), (h - 1, 0), (0, w - 1), (h // 2, w // 2)]
    for finest in (0, 1):
        for y, x in spots:
            img = rng.uniform(0, 255, (2, h, w)).astype(np.float32)
            img[1, y, x] = np.nan
            with pytest.raises(ValueError):
                st.build_pyramid(img, 2, finest=finest, second_derivatives=False,
                                 level0=finest == 0)


@pytest.mark.parametrize("B", [1, 5, 13])
def test_host_path_chunk_ramp_matches_device(torch, B):
    """The host-buffer pipeline's chunk schedule (1, 1, 2, 4, then up to 8
    pairs per chunk, each on its own stream) returns the device path's flows
    for every pair, eagerly and from the captured graph."""
    from paper_1603_03590_b200 import FlowEngine

    cfg = synth.CONFIGS["c1"]
    f1, f2 = synth.make_batch(cfg, seed=40, count=B, h=109, w=256)
    params = synth.dis_params(cfg, coarsest=3)
    eng = FlowEngine(B, 109, 256, params)
    want = eng.run(torch.from_numpy(f1).cuda(), torch.from_numpy(f2).cuda()).cpu().numpy()
    p1 = torch.from_numpy(f1).pin_memory()
    p2 = torch.from_numpy(f2).pin_memory()
    po = torch.empty((B, 109, 256, 2), dtype=torch.float64).pin_memory()
    for _ in range(3):  # eager, capture, replay
        po.zero_()
        eng.run_host(p1.numpy(), p2.numpy(), out=po.numpy())
        assert np.array_equal(po.numpy(), want)


def test_refinement_height_limit_is_a_documented_value_error(torch):
    """Variational refinement of a level taller than 2048 rows (16 cluster
    CTAs x 128 rows of the wavefront SOR) raises ValueError with the
    documented message instead of running; without
    refinement such levels run."""
    from paper_1603_03590_b200 import FlowEngine

    p = DisParams(patch_size=8, overlap=0.3, iterations=4, finest_scale=0, coarsest_scale=5,
                  variational=VarParams(outer_iters_fixed=1))
    with pytest.raises(ValueError, match="taller than 2048 rows"):
        FlowEngine(1, 2050, 256, p)
    q = dataclasses.replace(p, finest_scale=1)  # level 1 is 1025 rows: fine
    FlowEngine(1, 2050, 256, q)
    r = dataclasses.replace(p, variational=None)
    FlowEngine(1, 2050, 256, r)
