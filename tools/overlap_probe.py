"""Experiment: does splitting a c1 batch over concurrent streams, with the
later parts started a little after the first, hide the latency-bound coarse
levels under the throughput-bound fine levels?  Device-resident frames,
graph-replayed FlowEngine per part, stagger by a spin kernel
(torch.cuda._sleep) at the head of each later stream.  Prints ms per step
for each (parts, stagger) against the one-batch step.

usage: python tools/overlap_probe.py [--batch 64] [--steps 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1603_03590_b200 import FlowEngine  # noqa: E402
from tools import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--config", default="c1")
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    params = synth.dis_params(cfg)
    B = args.batch
    f1n, f2n = synth.make_batch(cfg, seed=0, count=B)
    dev = torch.device("cuda", 0)
    f1 = torch.from_numpy(np.ascontiguousarray(f1n)).to(dev)
    f2 = torch.from_numpy(np.ascontiguousarray(f2n)).to(dev)
    H, W = cfg.height, cfg.width
    clk_hz = torch.cuda.clock_rate() * 1e6 if hasattr(torch.cuda, "clock_rate") else 1.9e9

    def time_it(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        main = torch.cuda.current_stream()
        s.record(main)
        for _ in range(args.steps):
            fn()
        e.record(main)
        torch.cuda.synchronize()
        return s.elapsed_time(e) / args.steps

    ref_out = torch.empty((B, H, W, 2), dtype=torch.float64, device=dev)
    eng = FlowEngine(B, H, W, params, device=dev)
    st0 = torch.cuda.Stream(device=dev)

    def one():
        st0.wait_stream(torch.cuda.current_stream())
        eng.run(f1, f2, out=ref_out, stream=st0, check=False, graph=True)
        torch.cuda.current_stream().wait_stream(st0)

    base = time_it(one)
    print(f"one batch of {B}: {base:.3f} ms/step", flush=True)
    del eng
    for parts in (2, 4):
        nb = B // parts
        engs = [FlowEngine(nb, H, W, params, device=dev) for _ in range(parts)]
        outs = [torch.empty((nb, H, W, 2), dtype=torch.float64, device=dev) for _ in range(parts)]
        sts = [torch.cuda.Stream(device=dev) for _ in range(parts)]
        f1s = [f1[i * nb:(i + 1) * nb] for i in range(parts)]
        f2s = [f2[i * nb:(i + 1) * nb] for i in range(parts)]
        for stagger_us in (0, 200, 400, 700, 1000):
            cyc = int(stagger_us * 1e-6 * clk_hz)

            def split():
                cur = torch.cuda.current_stream()
                for i in range(parts):
                    sts[i].wait_stream(cur)
                    if i and cyc:
                        with torch.cuda.stream(sts[i]):
                            torch.cuda._sleep(cyc * i)
                    engs[i].run(f1s[i], f2s[i], out=outs[i], stream=sts[i], check=False,
                                graph=True)
                for i in range(parts):
                    cur.wait_stream(sts[i])

            t = time_it(split)
            same = all(torch.equal(outs[i], ref_out[i * nb:(i + 1) * nb]) for i in range(parts))
            print(f"{parts} parts, stagger {stagger_us} us x i: {t:.3f} ms/step "
                  f"({base / t:.3f}x) bit-identical={same}", flush=True)
        del engs, outs


if __name__ == "__main__":
    main()
