"""Randomised soak of the GPU path against the CPU oracle (test tooling, like
tests/: the oracle is only the checker).  Draws N random problems — level
sizes, batch, patch size / overlap / iterations / scales / downscale factor,
residual norm, mean normalisation, refinement weights / sweeps / outer
iterations, stereo and bidirectional mode, frame dtype, host or device entry
point — runs each through the C ABI and compares the flow with the oracle's
bit for bit.  Prints one line per failing case (with the seed to replay it)
and a summary.

    python tools/soak_parity.py [--cases 200] [--seed 0] [--max-px 40000]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_1603_03590_b200 import DisParams, FlowEngine, VarParams  # noqa: E402
from tools import synth  # noqa: E402


def draw_case(rng, max_px):
    ps = int(rng.choice([8, 8, 8, 12, 12, 4, 5, 9, 16]))
    down = int(rng.choice([2, 2, 2, 2, 3, 4]))
    finest = int(rng.choice([0, 1, 1, 2]))
    span = int(rng.integers(0, 4))
    coarsest = finest + span
    # the coarsest level must hold a patch (+ a few pixels)
    min_dim = (ps + int(rng.integers(1, 30))) * down ** coarsest
    h = min_dim + int(rng.integers(0, 40))
    w = min_dim + int(rng.integers(0, 120))
    while h * w > max_px and coarsest > finest:
        coarsest -= 1
        min_dim = (ps + 3) * down ** coarsest
        h = min_dim + int(rng.integers(0, 40))
        w = min_dim + int(rng.integers(0, 120))
    if h * w > max_px:
        s = (max_px / (h * w)) ** 0.5
        h = max(int(h * s), (ps + 2) * down ** coarsest)
        w = max(int(w * s), (ps + 2) * down ** coarsest)
    stereo = bool(rng.random() < 0.15)
    bidir = bool(not stereo and rng.random() < 0.15)
    refine = rng.random() < 0.8
    vp = None
    if refine:
        vp = VarParams(intensity_weight=float(rng.choice([5.0, 0.0, 2.5])),
                       gradient_weight=float(rng.choice([10.0, 0.0, 4.0])),
                       smoothness_weight=float(rng.choice([10.0, 1.0, 30.0])),
                       inner_sor_iters=int(rng.choice([5, 5, 1, 3, 8, 11])),
                       penalizer_eps=float(rng.choice([0.001, 0.01])),
                       sor_omega=float(rng.choice([1.6, 1.0, 1.9])),
                       outer_iters_fixed=(None if rng.random() < 0.3
                                          else int(rng.integers(1, 4))))
    norm = str(rng.choice(["l2", "l2", "l1", "huber"]))
    p = DisParams(patch_size=ps, overlap=float(rng.choice([0.0, 0.3, 0.4, 0.5, 0.75, 0.9])),
                  iterations=int(rng.choice([1, 4, 12, 32, 64])), finest_scale=finest,
                  coarsest_scale=coarsest, downscale=down,
                  use_mean_normalization=bool(rng.random() < 0.8), residual_norm=norm,
                  huber_b=float(rng.choice([1.0, 0.3, 4.0])), variational=vp,
                  mode="stereo" if stereo else "flow", bidirectional=bidir)
    batch = int(rng.choice([1, 1, 2, 3, 5]))
    dtype = rng.choice(["f32", "f32", "f64", "u8"])
    host = bool(rng.random() < 0.3)
    disp = float(rng.choice([0.5, 3.0, 8.0, 20.0]))
    return dict(h=int(h), w=int(w), params=p, batch=batch, dtype=str(dtype), host=host,
                stereo=stereo, disp=disp)


def draw_big_case(rng):
    """Batches whose finest level runs on the lane kernel (more than ~76k
    patches over the batch): work queue, padded query
    level, parked border windows and the straggler hand-off."""
    ps = int(rng.choice([8, 8, 12]))
    ov = float(rng.choice([0.5, 0.5, 0.75]))
    finest = int(rng.choice([0, 1]))
    coarsest = finest + int(rng.integers(1, 3))
    h = int(rng.integers(90, 230)) * (2 ** finest)
    w = int(rng.integers(180, 520)) * (2 ** finest)
    sp = max(1, int(ps * (1.0 - ov)))
    per_pair = ((h >> finest) // sp) * ((w >> finest) // sp)
    need = 80000  # > 148 * 2048 * 2 / 8 = 148 * 2048 * 4 / 16 patches
    batch = int(min(64, max(8, need // max(1, per_pair) + 2)))
    refine = rng.random() < 0.6
    vp = VarParams(outer_iters_fixed=1) if refine else None
    p = DisParams(patch_size=ps, overlap=ov, iterations=int(rng.choice([8, 32, 64])),
                  finest_scale=finest, coarsest_scale=coarsest,
                  use_mean_normalization=bool(rng.random() < 0.85),
                  residual_norm=str(rng.choice(["l2", "l2", "l1", "huber"])), variational=vp,
                  mode="flow")
    return dict(h=h, w=w, params=p, batch=batch, dtype="f32", host=bool(rng.random() < 0.2),
                stereo=False, disp=float(rng.choice([3.0, 10.0, 25.0])))


def run_case(c, seed):
    h, w, p, B = c["h"], c["w"], c["params"], c["batch"]
    f1 = np.empty((B, h, w), np.float32)
    f2 = np.empty((B, h, w), np.float32)
    for i in range(B):
        a, b, _ = synth.make_pair(seed * 16 + i, h, w, c["disp"], True, c["disp"])
        f1[i], f2[i] = a, b
    if c["dtype"] == "f64":
        f1, f2 = f1.astype(np.float64) * 1.0000001, f2.astype(np.float64) * 0.9999999
    elif c["dtype"] == "u8":
        f1, f2 = np.clip(f1, 0, 255).astype(np.uint8), np.clip(f2, 0, 255).astype(np.uint8)
    eng = FlowEngine(B, h, w, p, stereo=c["stereo"])
    if c["host"]:
        got = eng.run_host(f1, f2)
    else:
        got = eng.run(torch.from_numpy(f1).cuda(), torch.from_numpy(f2).cuda()).cpu().numpy()
    torch.cuda.synchronize()
    for i in range(B):
        fn = oracle.dis_stereo if c["stereo"] else oracle.dis_flow
        want = fn(f1[i], f2[i], p)
        if not np.array_equal(got[i], want):
            d = np.abs(got[i] - want)
            return f"pair {i}: max |d| {np.nanmax(d):.3e}, {int((d > 0).sum())} values differ"
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--max-px", type=int, default=40000)
    ap.add_argument("--only", type=int, default=-1, help="replay one case index")
    ap.add_argument("--big", action="store_true",
                    help="large batches whose finest level runs on the lane kernel")
    a = ap.parse_args()
    bad = skipped = 0
    stats = {"stereo": 0, "bidirectional": 0, "host": 0, "refined": 0, "pairs": 0, "pixels": 0}
    t0 = time.time()
    for k in range(a.cases):
        if a.only >= 0 and k != a.only:
            continue
        rng = np.random.default_rng([a.seed, k])
        c = draw_big_case(rng) if a.big else draw_case(rng, a.max_px)
        stats["stereo"] += c["stereo"]
        stats["bidirectional"] += c["params"].bidirectional
        stats["host"] += c["host"]
        stats["refined"] += c["params"].variational is not None
        stats["pairs"] += c["batch"]
        stats["pixels"] += c["batch"] * c["h"] * c["w"]
        tag = (f"case {k} (seed {a.seed}): {c['batch']}x{c['h']}x{c['w']} {c['dtype']} "
               f"{'host' if c['host'] else 'dev'} {c['params']}")
        try:
            msg = run_case(c, a.seed * 100003 + k)
        except (ValueError, RuntimeError, AssertionError) as exc:
            # both sides must refuse the same problems: ask the oracle too
            try:
                f = np.zeros((c["h"], c["w"]), np.float32)
                (oracle.dis_stereo if c["stereo"] else oracle.dis_flow)(f, f, c["params"])
                msg = f"GPU path raised {type(exc).__name__}: {exc} (the oracle accepts the problem)"
            except Exception:
                skipped += 1
                continue
        if msg:
            bad += 1
            print("MISMATCH", tag, "->", msg, flush=True)
    print(f"soak: {a.cases} cases, {bad} mismatches, {skipped} rejected by both sides, "
          f"{time.time() - t0:.0f} s; {stats}", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
