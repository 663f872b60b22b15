cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_ta.log 2>&1; tail -2 gpurun_out/pytest_ta.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --config c1 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value %.0f ms %.3f' % (d['value'], d['ms_per_step']), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
KERNELS="k_tensor_assemble:4 k_gradients_tile:0" bash tools/_exp_prof.sh e > /dev/null 2>&1
