"""The split host-buffer call (dis_flow_batch_host_async + dis_host_batch_finish,
FlowEngine.submit_host / finish_host): two calls in flight give the blocking
call's flow bit for bit, eagerly, while being captured and as replayed graphs;
errors surface at finish_host; an engine refuses a second call in flight."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1603_03590_b200 import DisParams, FlowEngine, VarParams  # noqa: E402
from tools import synth  # noqa: E402

pytestmark = pytest.mark.gpu


def _pairs(n, h, w, seed):
    f1 = np.empty((n, h, w), np.float32)
    f2 = np.empty((n, h, w), np.float32)
    for i in range(n):
        a, b, _ = synth.make_pair(seed + i, h, w, 6.0, True, 6.0)
        f1[i], f2[i] = a, b
    return f1, f2


def test_two_calls_in_flight_match_blocking_calls():
    h, w, n = 109, 256, 6
    params = DisParams(patch_size=8, overlap=0.5, iterations=32, finest_scale=1,
                       coarsest_scale=3, variational=VarParams(outer_iters_fixed=1))
    sets = [_pairs(n, h, w, 10), _pairs(n, h, w, 50)]
    ref_eng = FlowEngine(n, h, w, params)
    want = [ref_eng.run_host(a, b).copy() for a, b in sets]
    engs = [FlowEngine(n, h, w, params) for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    pins = [[torch.from_numpy(x).pin_memory().numpy() for x in s] for s in sets]
    outs = [torch.empty((n, h, w, 2), dtype=torch.float64).pin_memory().numpy() for _ in range(2)]
    for rnd in range(4):  # eager, capture, replay, replay
        for o in outs:
            o[...] = np.nan
        for k in range(2):
            engs[k].submit_host(pins[k][0], pins[k][1], outs[k], stream=streams[k])
        with pytest.raises(RuntimeError):
            engs[0].submit_host(pins[0][0], pins[0][1], outs[0], stream=streams[0])
        with pytest.raises(RuntimeError):
            engs[0].run_host(pins[0][0], pins[0][1])
        for k in (1, 0):
            got = engs[k].finish_host()
            assert got is outs[k]
            assert np.array_equal(got, want[k]), f"round {rnd} slot {k}"
    with pytest.raises(RuntimeError):
        engs[0].finish_host()


def test_pageable_buffers_and_error_at_finish():
    h, w, n = 64, 96, 2
    params = DisParams(patch_size=8, overlap=0.5, iterations=8, finest_scale=1,
                       coarsest_scale=2, variational=VarParams(outer_iters_fixed=1))
    f1, f2 = _pairs(n, h, w, 3)
    eng = FlowEngine(n, h, w, params)
    want = eng.run_host(f1, f2).copy()
    out = np.empty((n, h, w, 2))
    eng.submit_host(f1, f2, out)
    assert np.array_equal(eng.finish_host(), want)
    bad = f1.copy()
    bad[1, 5, 7] = np.nan
    eng.submit_host(bad, f2, out)
    with pytest.raises(ValueError, match="non-finite"):
        eng.finish_host()
    eng.submit_host(f1, f2, out)  # the engine is usable again
    assert np.array_equal(eng.finish_host(), want)


def test_float32_flow_out_is_the_rounded_float64_flow():
    """DIS_HOST_FLOW_F32: same computation, the flow rounded to nearest on the
    device (== astype(float32)); blocking, in flight and stereo."""
    h, w, n = 109, 256, 5
    params = DisParams(patch_size=8, overlap=0.5, iterations=32, finest_scale=1,
                       coarsest_scale=3, variational=VarParams(outer_iters_fixed=1))
    f1, f2 = _pairs(n, h, w, 21)
    eng = FlowEngine(n, h, w, params)
    want = eng.run_host(f1, f2).copy()
    out32 = np.empty((n, h, w, 2), np.float32)
    for _ in range(3):  # eager, captured (pageable: stays eager), repeated
        out32[...] = np.nan
        got = eng.run_host(f1, f2, out=out32)
        assert got is out32 and np.array_equal(out32, want.astype(np.float32))
    pin1, pin2 = (torch.from_numpy(x).pin_memory().numpy() for x in (f1, f2))
    pout = torch.empty((n, h, w, 2), dtype=torch.float32).pin_memory().numpy()
    for _ in range(3):  # pinned: eager, captured, replayed
        pout[...] = np.nan
        eng.submit_host(pin1, pin2, pout)
        assert np.array_equal(eng.finish_host(), want.astype(np.float32))
    # the float64 path on the same engine afterwards is untouched
    assert np.array_equal(eng.run_host(f1, f2), want)
    seng = FlowEngine(n, h, w, params, stereo=True)
    swant = seng.run_host(f1, f2).copy()
    assert np.array_equal(seng.run_host(f1, f2, out=out32), swant.astype(np.float32))
    with pytest.raises(ValueError):
        eng.run_host(f1, f2, out=np.empty((n, h, w, 2), np.float16))
