cd $GRAFT_REPO_ROOT
LBG_K12_TWO=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -m gpu -q -x -k "coupled or setu or fused or sweep or particle_bed or decomposition_invariance or config5 or mapping" > gpurun_out/r02_g17_pytest_two.log 2>&1; echo rc=$? >> gpurun_out/r02_g17_pytest_two.log
for env in "LBG_K12_TWO=1" "LBG_K12_TWO=0" "LBG_K12_TWO=1" "LBG_K12_TWO=0"; do
  env $env AB_STEPS=30 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_g17_ab.log 2>&1
done
