cd $GRAFT_REPO_ROOT
for P in 1 2 3; do DIS_SOR_P=$P timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_p$P.log 2>&1; echo "P=$P $(tail -1 gpurun_out/pytest_p$P.log)"; done
for cfg in "1 32 512" "64 218 512" "148 128 512"; do
  for K in "DIS_SOR_ROWS=0" "DIS_SOR_P=1" "DIS_SOR_P=2" "DIS_SOR_P=3"; do
    echo "$K $(env $K timeout 120 python tools/sor_bench.py $cfg 5 2>&1 | tail -1)"
  done
done
