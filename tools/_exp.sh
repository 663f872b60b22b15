# ad-hoc GPU experiments (env knobs of the kernels); output in gpurun_out/exp.log
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --config ${CFG:-c1}"
run() { echo "== $1" >> gpurun_out/exp.log; env $1 $B 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value %.0f ms %.3f' % (d['value'], d['ms_per_step']), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" >> gpurun_out/exp.log 2>&1; }
rm -f gpurun_out/exp.log
for v in $KNOBS; do run "$v"; done
cat gpurun_out/exp.log
