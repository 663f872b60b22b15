cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_cfg.log 2>&1; tail -2 gpurun_out/pytest_cfg.log
for c in c1 c0 c2 c3 c4; do
  STEPS=20; [ $c = c3 ] && STEPS=5; [ $c = c4 ] && STEPS=3; [ $c = c2 ] && STEPS=10
  timeout 900 python bench.py --steps $STEPS --warmup 3 --config $c --cpu-pairs 16 > gpurun_out/bench_cfg_$c.log 2>&1
  tail -1 gpurun_out/bench_cfg_$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$c', 'value %.1f ms %.3f' % (d['value'], d['ms_per_step']), 'e2e', round(d['e2e']['value'],1) if d.get('e2e') else None, 'cpu', round(d['cpu_baseline']['value'],2) if d.get('cpu_baseline') else None, {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" 2>&1 | tail -1
done
