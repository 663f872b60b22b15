# ad-hoc GPU experiments (env knobs of the kernels); output in gpurun_out/exp_*.log
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --config c1"
run() { echo "== $1" >> gpurun_out/exp.log; env $1 $B 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value %.0f ms %.3f' % (d['value'], d['ms_per_step']), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" >> gpurun_out/exp.log 2>&1; }
run "X=0"
run "DIS_SOR_RT=2"
run "DIS_SOR_RT=4"
run "DIS_GROUP_LANES=400000"
run "DIS_GROUP_LANES=2000000"
run "DIS_GROUP_LANES=0"
(cd tools/micro && ./tput) > gpurun_out/tput.log 2>&1
