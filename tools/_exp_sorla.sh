cd $GRAFT_REPO_ROOT
L=paper_1603_03590_b200/libdis_b200.so
cp $L /tmp/orig.so
for so in exp_so/la5.so exp_so/la8.so exp_so/la12.so; do
  cp $so $L
  for cfg in "1 32 512" "64 218 512" "148 128 512"; do
    echo "$so $(DIS_SOR_P=2 timeout 120 python tools/sor_bench.py $cfg 5 2>&1 | tail -1)"
  done
done
cp /tmp/orig.so $L
