#!/bin/bash
# One GPU session: parity tests, bench, ncu launch list + full captures.
# usage: tools/gpu_round.sh <tag> [config]
set -u
TAG=${1:-r}
CFG=${2:-c1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/smi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rfE > $OUT/pytest_gpu_$TAG.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 --config $CFG > $OUT/bench_$TAG.log 2>&1
PROF="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config $CFG"
if [ "${NCU:-1}" = "1" ]; then
  $PROF > $OUT/prof_plain_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $PROF > $OUT/ncu_launch_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_sor|k_patch_search" -s 8 -c 2 -o $OUT/prof_$TAG -f $PROF > $OUT/ncu_full_$TAG.log 2>&1
fi
echo finished
