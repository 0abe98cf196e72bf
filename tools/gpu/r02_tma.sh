cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest -x -q tests/test_gpu_variants.py -k "K12_TMA" > gpurun_out/r02_tma2_pytest.log 2>&1
LBG_K12_TMA=1 LBG_K12=2 timeout 900 python -m pytest -x -q tests/test_gpu_fullsize.py -k "config3 or bed" >> gpurun_out/r02_tma2_pytest.log 2>&1
for env in "LBG_K12=2" "LBG_K12=2 LBG_K12_TMA=1" "LBG_K12=2" "LBG_K12=2 LBG_K12_TMA=1"; do
  env $env AB_STEPS=30 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_tma2_ab.log 2>&1
done
LBG_K12=2 LBG_K12_TMA=1 AB_STEPS=5 timeout 600 ncu --set full --clock-control none --import-source on -k regex:coupled_tma -c 1 -o gpurun_out/r02_tma2 -f python tests/ab_coupled_sweep.py > gpurun_out/r02_tma2_ncu.log 2>&1
