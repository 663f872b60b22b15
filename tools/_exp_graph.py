"""Experiment: eager FlowEngine.run vs a CUDA-graph replay of the same call."""
import sys
import torch
sys.path.insert(0, '.')
from paper_1603_03590_b200 import FlowEngine
from tools import synth
import bench

for name in sys.argv[1:] or ['c0']:
    cfg = synth.CONFIGS[name]
    params = synth.dis_params(cfg)
    B = cfg.batch
    f1n, f2n = bench.make_inputs(cfg, seed=0, count=B, workers=16)
    f1 = torch.from_numpy(f1n).cuda(); f2 = torch.from_numpy(f2n).cuda()
    out = torch.empty((B, cfg.height, cfg.width, 2), dtype=torch.float64, device='cuda')
    eng = FlowEngine(B, cfg.height, cfg.width, params)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            eng.run(f1, f2, out=out, stream=s, check=False)
    torch.cuda.synchronize()
    ref = out.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        eng.run(f1, f2, out=out, stream=s, check=False)
    torch.cuda.synchronize()
    out.zero_(); g.replay(); torch.cuda.synchronize()
    same = torch.equal(out, ref)
    def t(fn, n):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        fn(); torch.cuda.synchronize()
        e0.record(s)
        for _ in range(n): fn()
        e1.record(s); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n
    n = 200 if name == 'c0' else 20
    with torch.cuda.stream(s):
        te = t(lambda: eng.run(f1, f2, out=out, stream=s, check=False), n)
        tg = t(lambda: g.replay(), n)
    print(name, 'eager %.3f ms graph %.3f ms same=%s' % (te, tg, same), flush=True)
