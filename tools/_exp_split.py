"""Experiment: a batch split over S concurrent streams (S engines of B/S
pairs) vs one engine of B pairs; prints pairs/s per split."""
import sys
import torch
sys.path.insert(0, '.')
from paper_1603_03590_b200 import FlowEngine
from tools import synth
import bench

name = sys.argv[1] if len(sys.argv) > 1 else 'c1'
cfg = synth.CONFIGS[name]
params = synth.dis_params(cfg)
B = cfg.batch
f1n, f2n = bench.make_inputs(cfg, seed=0, count=B, workers=16)
f1 = torch.from_numpy(f1n).cuda()
f2 = torch.from_numpy(f2n).cuda()
out = torch.empty((B, cfg.height, cfg.width, 2), dtype=torch.float64, device='cuda')
for S in (1, 2, 4):
    b = B // S
    engs = [FlowEngine(b, cfg.height, cfg.width, params) for _ in range(S)]
    sts = [torch.cuda.Stream() for _ in range(S)]
    def step():
        ev = torch.cuda.current_stream().record_event()
        for i in range(S):
            sts[i].wait_event(ev)
            engs[i].run(f1[i*b:(i+1)*b], f2[i*b:(i+1)*b], out=out[i*b:(i+1)*b], stream=sts[i], check=False)
        for i in range(S):
            torch.cuda.current_stream().wait_stream(sts[i])
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        step()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(name, 'S', S, 'ms/step %.3f' % ms, 'pairs/s %.0f' % (B / ms * 1e3), flush=True)
    del engs
    torch.cuda.empty_cache()
