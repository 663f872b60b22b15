cd $GRAFT_REPO_ROOT
for cfg in "1 128 512" "64 128 512" "148 128 512" "64 218 512" "64 64 512"; do
  for K in "DIS_SOR_ROWS=0" "DIS_SOR_P=1" "DIS_SOR_P=2" "DIS_SOR_P=5"; do
    echo "$K $(env $K timeout 120 python tools/sor_bench.py $cfg 5 2>&1 | tail -1)"
  done
done
