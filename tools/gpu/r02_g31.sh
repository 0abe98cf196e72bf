cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -m gpu -q -x > gpurun_out/r02_g31_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_g31_pytest.log
LBG_K12=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -m gpu -q -x > gpurun_out/r02_g31_pytest_list.log 2>&1; echo rc=$? >> gpurun_out/r02_g31_pytest_list.log
for env in "LBG_K12=1" "LBG_K12=2" "LBG_K12=3" "LBG_K12=0"; do
  env $env AB_STEPS=20 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_g31_ab3.log 2>&1
  env $env timeout 400 python tests/ab_config5_sweep.py >> gpurun_out/r02_g31_ab5.log 2>&1
done
