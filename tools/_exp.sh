cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for i in 1 2; do timeout 60 python tools/sor_bench.py 16 436 1024 3; done
timeout 60 python tools/sor_bench.py 64 218 512 5
timeout 60 python tools/sor_bench.py 64 109 256 5
