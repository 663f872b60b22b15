cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "refine or end_to_end or batched" > gpurun_out/pytest_sorx.log 2>&1; tail -2 gpurun_out/pytest_sorx.log
for cfg in "64 218 512" "64 109 256" "64 54 128"; do
  for C in 1 2; do
    DIS_SOR_CLUSTER=$C timeout 120 python tools/sor_bench.py $cfg 5 2>&1 | tail -1
  done
done > gpurun_out/sor_sweep.log 2>&1
cat gpurun_out/sor_sweep.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --config c1 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value %.0f ms %.3f' % (d['value'], d['ms_per_step']), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
