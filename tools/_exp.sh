cd $GRAFT_REPO_ROOT
PROF="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config c1"
$PROF > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_patch_gn|k_patch_prep" -s 8 -c 2 -o gpurun_out/psprof -f $PROF > gpurun_out/psprof_ncu.log 2>&1
