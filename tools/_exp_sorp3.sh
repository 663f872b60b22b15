cd $GRAFT_REPO_ROOT
for cfg in "148 32 512" "74 64 512" "1 32 512" "1 64 512"; do
  for K in "DIS_SOR_ROWS=0" "DIS_SOR_P=2"; do
    echo "$K $(env $K timeout 120 python tools/sor_bench.py $cfg 5 2>&1 | tail -1)"
  done
done
for C in 1 2; do echo "C=$C $(DIS_SOR_CLUSTER=$C DIS_SOR_ROWS=0 timeout 120 python tools/sor_bench.py 1 64 512 5 2>&1 | tail -1)"; done
