cd $GRAFT_REPO_ROOT
L=paper_1603_03590_b200/libdis_b200.so
cp $L /tmp/orig.so
for so in exp_so/tr0.so exp_so/tr160.so; do
  cp $so $L
  for cfg in "1 32 512" "64 218 512"; do
    echo "$so $cfg P=1: $(DIS_SOR_P=1 timeout 120 python tools/_exp_trace.py $cfg 2>&1 | tail -1)"
  done
done
cp /tmp/orig.so $L
for P in 1 2; do DIS_SOR_P=$P timeout 300 python -m pytest tests -m gpu -x -q -k "refine or flow or stereo or sor" > gpurun_out/pytest_tr.log 2>&1; echo "P=$P $(tail -1 gpurun_out/pytest_tr.log)"; done
for cfg in "1 32 512" "64 218 512" "148 128 512"; do
  for K in "DIS_SOR_P=1" "DIS_SOR_P=2"; do
    echo "$K $(env $K timeout 120 python tools/sor_bench.py $cfg 5 2>&1 | tail -1)"
  done
done
