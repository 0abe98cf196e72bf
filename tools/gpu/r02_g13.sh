cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_aa.py tests/test_gpu_parity.py tests/test_dropin.py -m gpu -q -x > gpurun_out/r02_g13_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_g13_pytest.log
for env in "LBG_K12=1" "LBG_K12_PIPE=1" "LBG_K12=0" "LBG_WALK_MINB=5" "LBG_K12=1" "LBG_K12_PIPE=1"; do
  env $env AB_REDUCE=1 AB_STEPS=30 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_g13_ab.log 2>&1
done
LBG_K12_PIPE=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -m gpu -q -x -k "coupled or setu or fused or sweep or particle_bed or decomposition_invariance or config5" > gpurun_out/r02_g13_pytest_pipe.log 2>&1; echo rc=$? >> gpurun_out/r02_g13_pytest_pipe.log
timeout 3000 python -m pytest tests/test_gpu_checked.py -m gpu -q -x > gpurun_out/r02_g13_checked.log 2>&1; echo rc=$? >> gpurun_out/r02_g13_checked.log
