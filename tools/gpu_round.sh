#!/bin/bash
# One GPU session: smoke, parity tests, bench, ncu launch list + full capture
# of every kernel of one pipeline step.
# usage: tools/gpu_round.sh <tag> [config]
set -u
TAG=${1:-r}
CFG=${2:-c1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/smi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rfE > $OUT/pytest_gpu_$TAG.log 2>&1
fi
timeout 900 python bench.py --steps 20 --warmup 3 --config $CFG > $OUT/bench_$TAG.log 2>&1
PROF="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-c3 --config $CFG"
if [ "${NCU:-1}" = "1" ]; then
  $PROF > $OUT/prof_plain_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $PROF > $OUT/ncu_launch_$TAG.log 2>&1
  # one full pipeline step (the second warm-up step) — every kernel once
  NL=$(python -c "import json,sys; d=json.loads(open('$OUT/prof_plain_$TAG.log').read().strip().splitlines()[-1]); print(int(d['gpu_launches']))")
  ncu --set full --clock-control none --import-source on -k regex:"^k_" -s $NL -c $NL -o /tmp/full_$TAG -f $PROF > $OUT/ncu_full_$TAG.log 2>&1
  ncu -i /tmp/full_$TAG.ncu-rep --page raw --csv > $OUT/full_raw_$TAG.csv 2>/dev/null
  ncu -i /tmp/full_$TAG.ncu-rep --page details --csv > $OUT/full_details_$TAG.csv 2>/dev/null
  # the report itself only when it fits gpurun's 64 MiB copy-back
  SZ=$(stat -c %s /tmp/full_$TAG.ncu-rep 2>/dev/null || echo 0)
  if [ "$SZ" -lt 40000000 ]; then cp /tmp/full_$TAG.ncu-rep $OUT/; fi
  # the top kernels' source/SASS pages (hot lines)
  # (name:skip — the finest level's launch of the first warm-up step)
  for KS in k_sor:4 k_patch_gn:0 k_tensor_assemble:4 k_patch_gn_group:3 k_densify:4; do
    K=${KS%%:*}; S=${KS##*:}
    ncu --set full --clock-control none --import-source on -k regex:"^$K(<.*)?$" -s $S -c 1 -o /tmp/src_$K -f $PROF > /dev/null 2>&1
    ncu -i /tmp/src_$K.ncu-rep --page source --csv --print-source sass > $OUT/sass_${K}_$TAG.csv 2>/dev/null
  done
fi
echo finished
