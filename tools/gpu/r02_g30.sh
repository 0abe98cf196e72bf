cd $GRAFT_REPO_ROOT
for env in "LBG_K12=1" "LBG_K12=0" "LBG_K12_PIPE=0" "LBG_K12=0 LBG_K2_CONCURRENT=0"; do
  env $env timeout 400 python tests/ab_config5_sweep.py >> gpurun_out/r02_g30_ab.log 2>&1
done
AB_STEPS=3 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g30_launches.csv python tests/ab_config5_sweep.py > /dev/null 2>&1
LBG_K12=0 AB_STEPS=3 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g30_launches_split.csv python tests/ab_config5_sweep.py > /dev/null 2>&1
