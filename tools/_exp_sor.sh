cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_known_answers_gpu.py -q -x -k "refine or end_to_end or batched or sweep" > gpurun_out/pytest_sorx.log 2>&1; tail -1 gpurun_out/pytest_sorx.log
for cfg in "64 218 512" "64 109 256" "64 54 128"; do
  timeout 120 python tools/sor_bench.py $cfg 5 2>&1 | tail -1
done
KNOBS="X=0" bash tools/_exp.sh
