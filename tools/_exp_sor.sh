cd $GRAFT_REPO_ROOT
for cfg in "64 218 512" "128 218 512" "256 540 960"; do
  for C in 0 2 3 4 5 8 9; do
    DIS_SOR_CLUSTER=$C timeout 120 python tools/sor_bench.py $cfg 3 2>&1 | tail -1
  done
done
