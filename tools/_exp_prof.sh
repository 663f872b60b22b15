# source-level ncu captures of the top kernels (finest-level launch of warm-up step 1)
cd $GRAFT_REPO_ROOT
TAG=${1:-x}
PROF="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --config c1"
for KS in ${KERNELS:-k_sor:4 k_patch_gn:0 k_patch_gn_group:3}; do
  K=${KS%%:*}; S=${KS##*:}
  ncu --set full --clock-control none --import-source on -k regex:"^$K(<.*)?$" -s $S -c 1 -o /tmp/src_$K -f $PROF > /dev/null 2>&1
  ncu -i /tmp/src_$K.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_${K}_$TAG.csv 2>/dev/null
  ncu -i /tmp/src_$K.ncu-rep --page raw --csv > gpurun_out/raw_${K}_$TAG.csv 2>/dev/null
done
ls -la gpurun_out | tail -8
