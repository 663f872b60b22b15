cd $GRAFT_REPO_ROOT
export DIS_SOR_RT=1
python tools/sor_bench.py 16 54 128 2 > gpurun_out/sorprof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sor -s 1 -c 1 -o gpurun_out/sorprof6 -f python tools/sor_bench.py 16 54 128 2 > gpurun_out/sorprof_ncu.log 2>&1
