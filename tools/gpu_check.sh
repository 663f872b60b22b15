#!/bin/bash
# One GPU session for a code change: host description, smoke, GPU tests,
# the reference arm and the default bench line.
# usage: tools/gpu_check.sh <tag> [pytest -k expr]
set -u
TAG=${1:-chk}
K=${2:-}
OUT=gpurun_out
mkdir -p $OUT
( nproc; lscpu | head -20; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv ) > $OUT/host_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
if [ "${TESTS:-1}" = "1" ]; then
  if [ -n "$K" ]; then
    timeout 2400 python -m pytest tests -m gpu -q -rfE -k "$K" > $OUT/pytest_gpu_$TAG.log 2>&1
  else
    timeout 2400 python -m pytest tests -m gpu -q -rfE > $OUT/pytest_gpu_$TAG.log 2>&1
  fi
  echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu_$TAG.log
fi
if [ "${REF:-1}" = "1" ]; then
  timeout 900 python bench.py --impl reference --steps ${REF_STEPS:-5} --warmup 1 > $OUT/ref_$TAG.log 2>&1; echo "ref rc=$?"
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout 1200 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS:-} > $OUT/bench_$TAG.log 2>&1; echo "bench rc=$?"
fi
echo finished
