"""Experiment: e2e (host-buffer path) time of c1 pairs for batch sizes 1..64
(graph-replayed after two calls), to separate the pipeline head from the
steady state:  python tools/e2e_scaling.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1603_03590_b200 import FlowEngine
from tools import synth

cfg = synth.CONFIGS["c1"]
f1, f2 = synth.make_batch(cfg, seed=0, count=8)
for B in (1, 2, 4, 8, 16, 32, 64):
    a = np.concatenate([f1] * 8)[:B]
    b = np.concatenate([f2] * 8)[:B]
    eng = FlowEngine(B, cfg.height, cfg.width, synth.dis_params(cfg))
    p1 = torch.from_numpy(a).pin_memory()
    p2 = torch.from_numpy(b).pin_memory()
    po = torch.empty((B, cfg.height, cfg.width, 2), dtype=torch.float64).pin_memory()
    for _ in range(3):
        eng.run_host(p1.numpy(), p2.numpy(), out=po.numpy())
    torch.cuda.synchronize()
    n = 10
    t = time.perf_counter()
    for _ in range(n):
        eng.run_host(p1.numpy(), p2.numpy(), out=po.numpy())
    dt = (time.perf_counter() - t) / n
    d1 = torch.from_numpy(a).cuda()
    d2 = torch.from_numpy(b).cuda()
    do = torch.empty((B, cfg.height, cfg.width, 2), dtype=torch.float64, device="cuda")
    for _ in range(2):
        eng.run(d1, d2, out=do)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        eng.run(d1, d2, out=do)
    torch.cuda.synchronize()
    dd = (time.perf_counter() - t) / n
    mb = B * cfg.height * cfg.width * (8 + 16) / 1e6
    print(f"B={B:3d}: e2e {dt * 1e3:7.3f} ms ({B / dt:6.0f} pairs/s), device (eager) {dd * 1e3:7.3f} ms, "
          f"copies {mb:6.1f} MB", flush=True)
    del eng
