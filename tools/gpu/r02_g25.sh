cd $GRAFT_REPO_ROOT
AB_REDUCE=1 AB_STEPS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"map_warp|walk_chain" -c 2 -o gpurun_out/r02_mapwalk2 python tests/ab_coupled_sweep.py > /dev/null 2>&1
