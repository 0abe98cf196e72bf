cd $GRAFT_REPO_ROOT
for env in "LBG_K12=3" "LBG_K12=3 LBG_K12_SPLIT_CONC=1" "LBG_K12=2" "LBG_K12=3 LBG_K12_SPLIT_CONC=1"; do
  env $env AB_STEPS=20 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_g32_ab3.log 2>&1
  env $env timeout 400 python tests/ab_config5_sweep.py >> gpurun_out/r02_g32_ab5.log 2>&1
done
