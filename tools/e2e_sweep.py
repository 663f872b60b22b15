"""Experiment: e2e (host-buffer path) step time of c1 for chunk schedules
(DIS_HOST_CHUNKS=n equal chunks, unset = the ramp).  Run once per setting:
python tools/e2e_sweep.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1603_03590_b200 import FlowEngine
from tools import synth

cfg = synth.CONFIGS["c1"]
B = 64
f1, f2 = synth.make_batch(cfg, seed=0, count=8)
f1 = np.concatenate([f1] * 8)
f2 = np.concatenate([f2] * 8)
eng = FlowEngine(B, cfg.height, cfg.width, synth.dis_params(cfg))
p1 = torch.from_numpy(f1).pin_memory()
p2 = torch.from_numpy(f2).pin_memory()
po = torch.empty((B, cfg.height, cfg.width, 2), dtype=torch.float64).pin_memory()
for _ in range(3):
    eng.run_host(p1.numpy(), p2.numpy(), out=po.numpy())
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    eng.run_host(p1.numpy(), p2.numpy(), out=po.numpy())
dt = (time.perf_counter() - t) / 10
d = torch.empty(po.shape, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    po.copy_(d, non_blocking=True)
torch.cuda.synchronize()
d2h = (time.perf_counter() - t) / 5
print(f"chunks={os.environ.get('DIS_HOST_CHUNKS', 'ramp')}: e2e {dt * 1e3:.2f} ms "
      f"({B / dt:.0f} pairs/s); D2H of the flow alone {d2h * 1e3:.2f} ms", flush=True)
