cd $GRAFT_REPO_ROOT
for spec in "256 540 960:0 5 9" "256 270 480:0 3 5" "256 135 240:0 2 3" "31 1080 1920:0 9 12 16" "31 540 960:0 5 9" "64 218 512:0 2 4"; do
  cfg=${spec%%:*}; Cs=${spec##*:}
  for C in $Cs; do
    echo "C=$C $(DIS_SOR_CLUSTER=$C timeout 120 python tools/sor_bench.py $cfg 3 2>&1 | tail -1)"
  done
done
