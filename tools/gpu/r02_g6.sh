cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py tests/test_gpu_reference_cases.py -m gpu -q -x > gpurun_out/r02_g6_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_g6_pytest.log
LBG_K12_LR=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -m gpu -q -x -k "coupled or setu or fused or mapping_and_solid or sweep or particle_bed or decomposition_invariance" > gpurun_out/r02_g6_pytest_lr.log 2>&1; echo rc=$? >> gpurun_out/r02_g6_pytest_lr.log
for env in "LBG_K12=1" "LBG_DIRECT_INDEX=0" "LBG_K12_LR=1" "LBG_K12_LR=1 LBG_K12_LR_SM=6" "LBG_K12_LR=1 LBG_K12_LR_SM=8" "LBG_K12_LR=1 LBG_K12_LR_SM=5" "LBG_K12=1"; do
  env $env AB_STEPS=30 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_g6_ab.log 2>&1
done
PROBE_STEPS=3 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g6_launches.csv python tests/coupled_probe.py scratch > /dev/null 2>&1
