cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
PROF="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config c1"
$PROF > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $PROF > gpurun_out/ncu_launch.log 2>&1
