cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/exp_pytest.log 2>&1
tail -3 gpurun_out/exp_pytest.log
PROF="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config c1"
$PROF > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_exp.csv $PROF > gpurun_out/ncu_launch_exp.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --config c1 > gpurun_out/bench_exp.log 2>&1
tail -1 gpurun_out/bench_exp.log | cut -c1-400
