# time prebuilt library variants (exp_so/*.so, swapped in place); output in gpurun_out/exp_so.log
cd $GRAFT_REPO_ROOT
L=paper_1603_03590_b200/libdis_b200.so
cp $L /tmp/orig.so
rm -f gpurun_out/exp_so.log
for so in ${SOS:-exp_so/*.so}; do
  cp $so $L
  for cfg in ${CFGS:-c1}; do
    echo "== $so $cfg" >> gpurun_out/exp_so.log
    python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --config $cfg 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value %.0f ms %.3f' % (d['value'], d['ms_per_step']), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" >> gpurun_out/exp_so.log 2>&1
  done
done
cp /tmp/orig.so $L
cat gpurun_out/exp_so.log
