cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_exp5.log 2>&1; tail -2 gpurun_out/pytest_exp5.log
bash tools/knob_sweep.sh e5 c1 20 "g64|DIS_B200_LIB=exp_so/libdis_g64.so" "t256|X=1"
bash tools/knob_sweep.sh e5c3 c3 5 "t256|X=1"
