cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
python tools/sor_bench.py 64 218 512 5
python tools/sor_bench.py 16 436 1024 3
python tools/sor_bench.py 64 54 128 5
python tools/sor_bench.py 64 109 256 5
