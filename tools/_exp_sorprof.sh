# source-level ncu capture of the SOR kernel of tools/sor_bench.py (single CTA case)
cd $GRAFT_REPO_ROOT
for K in "DIS_SOR_ROWS=0:old" "DIS_SOR_P=2:p2"; do
  KV=${K%%:*}; T=${K##*:}
  env $KV ncu --set full --clock-control none --import-source on -k regex:"k_sor" -s 1 -c 1 -o /tmp/sorp_$T -f python tools/sor_bench.py ${CFG:-1 32 512} 2 > /dev/null 2>&1
  ncu -i /tmp/sorp_$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_sorb_$T.csv 2>/dev/null
  ncu -i /tmp/sorp_$T.ncu-rep --page raw --csv > gpurun_out/raw_sorb_$T.csv 2>/dev/null
done
ls -la gpurun_out | tail -4
