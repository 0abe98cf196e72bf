cd $GRAFT_REPO_ROOT
AB_REDUCE=1 AB_STEPS=3 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g14_launches.csv python tests/ab_coupled_sweep.py > /dev/null 2>&1
AB_REDUCE=1 LBG_WALK_MINB=5 AB_STEPS=3 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g14_launches5.csv python tests/ab_coupled_sweep.py > /dev/null 2>&1
AB_REDUCE=1 AB_STEPS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_chain -s 1 -c 1 -o gpurun_out/r02_walk2 python tests/ab_coupled_sweep.py > /dev/null 2>&1
AB_STEPS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:unified_pipe -s 3 -c 1 -o gpurun_out/r02_pipe python tests/ab_coupled_sweep.py > /dev/null 2>&1
