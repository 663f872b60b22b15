#!/bin/bash
# Kernel-class times of one config under several library variants / env knobs
# (device-resident pass only).  Each case: "<label>|<env assignments>".
# usage: tools/knob_sweep.sh <tag> <config> <steps> "<label>|<env>" ...
set -u
TAG=$1; CFG=$2; STEPS=$3; shift 3
OUT=gpurun_out
mkdir -p $OUT
for CASE in "$@"; do
  LABEL=${CASE%%|*}; ENVS=${CASE#*|}
  env $ENVS timeout 600 python bench.py --steps $STEPS --warmup 3 --config $CFG --no-e2e --no-cpu --no-c3 \
    > $OUT/sweep_${TAG}_${LABEL}.log 2>&1
  tail -1 $OUT/sweep_${TAG}_${LABEL}.log | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read())
    print('$LABEL', '%.3f ms/step' % d['ms_per_step'], {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})
except Exception as e:
    print('$LABEL', 'failed', e)"
done
