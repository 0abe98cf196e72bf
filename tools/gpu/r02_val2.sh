cd $GRAFT_REPO_ROOT
LBG_REDUCE_PROFILE=1 AB_REDUCE=1 AB_STEPS=10 timeout 600 python tests/ab_coupled_sweep.py > gpurun_out/r02_val2_reduce.log 2>&1
timeout 5400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_val2_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_val2_pytest.log
