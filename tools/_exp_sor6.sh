cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -rfE > gpurun_out/pytest_sor8.log 2>&1; tail -5 gpurun_out/pytest_sor6.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --config c1 > gpurun_out/bench_sor8.log 2>&1
tail -1 gpurun_out/bench_sor8.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value %.0f ms %.3f' % (d['value'], d['ms_per_step']), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
PROF="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config c1"
ncu --set full --clock-control none --import-source on -k regex:"^k_sor(<.*)?$" -s 4 -c 1 -o /tmp/sor6 -f $PROF > /dev/null 2>&1
ncu -i /tmp/sor6.ncu-rep --page raw --csv > gpurun_out/sor8_raw.csv 2>/dev/null
ncu -i /tmp/sor6.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/sor8_src.csv 2>/dev/null
ncu --set full --clock-control none -k regex:"^k_tensor_assemble$" -s 4 -c 1 -o /tmp/ta6 -f $PROF > /dev/null 2>&1
ncu -i /tmp/ta6.ncu-rep --page raw --csv > gpurun_out/ta8_raw.csv 2>/dev/null
