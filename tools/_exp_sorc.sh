cd $GRAFT_REPO_ROOT
for cfg in "64 218 512" "64 109 256"; do
  for C in 0 2 3 4; do
    echo "C=$C $(DIS_SOR_CLUSTER=$C timeout 120 python tools/sor_bench.py $cfg 5 2>&1 | tail -1)"
  done
done
