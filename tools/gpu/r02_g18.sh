cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py tests/test_gpu_aa.py -m gpu -q -x > gpurun_out/r02_g18_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_g18_pytest.log
for env in "LBG_K12_NOWRAP=1" "LBG_K12_NOWRAP=0" "LBG_K12_TWO=0" "LBG_K12_NOWRAP=1" "LBG_K12_NOWRAP=0" "LBG_K12_TWO=0"; do
  env $env AB_STEPS=30 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_g18_ab.log 2>&1
done
AB_STEPS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:unified_pipe -s 3 -c 1 -o gpurun_out/r02_pipe4 python tests/ab_coupled_sweep.py > /dev/null 2>&1
