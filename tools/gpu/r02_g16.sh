cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -m gpu -q -x > gpurun_out/r02_g16_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_g16_pytest.log
for env in "LBG_K12_PIPE=1" "LBG_K12_PIPE=0" "LBG_K12_PIPE=1" "LBG_K12_PIPE=0"; do
  env $env AB_STEPS=30 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_g16_ab.log 2>&1
done
AB_STEPS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:unified_pipe -s 3 -c 1 -o gpurun_out/r02_pipe3 python tests/ab_coupled_sweep.py > /dev/null 2>&1
