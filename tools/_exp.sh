cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_exp15.log 2>&1; tail -1 gpurun_out/pytest_exp15.log
bash tools/knob_sweep.sh e15 c1 20 "tma|X=1"
bash tools/knob_sweep.sh e15c4 c4 3 "tma|X=1"
bash tools/knob_sweep.sh e15c2 c2 10 "tma|X=1"
