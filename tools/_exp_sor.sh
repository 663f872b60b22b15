cd $GRAFT_REPO_ROOT
for cfg in "256 270 480" "256 135 240" "64 109 256" "31 540 960"; do
  for C in 0 3 5 9 16; do
    DIS_SOR_CLUSTER=$C timeout 120 python tools/sor_bench.py $cfg 3 2>&1 | tail -1
  done
done
