timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_hg.log 2>&1; tail -1 gpurun_out/pytest_hg.log
for g in 0 1; do for c in c1 c0 c3; do echo "HG=$g $c $(DIS_HOST_GRAPH=$g timeout 300 python bench.py --steps 10 --warmup 3 --config $c --no-cpu --e2e-steps 10 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'e2e', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],3))")"; done; done
