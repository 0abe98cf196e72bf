cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_aa.py tests/test_gpu_parity.py tests/test_dropin.py -m gpu -q -x > gpurun_out/r02_g11_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_g11_pytest.log
for env in "LBG_K12=1" "LBG_K12_PIPE=1" "LBG_K12_SM=4" "LBG_K12=0" "LBG_K12=1"; do
  env $env AB_STEPS=30 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_g11_ab.log 2>&1
done
timeout 300 python tests/ab_config2_variants.py >> gpurun_out/r02_g11_ab.log 2>&1
timeout 3000 python -m pytest tests/test_gpu_checked.py -m gpu -q -x > gpurun_out/r02_g11_checked.log 2>&1; echo rc=$? >> gpurun_out/r02_g11_checked.log
