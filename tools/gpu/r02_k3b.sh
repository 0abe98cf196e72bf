cd $GRAFT_REPO_ROOT
AB_MAPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:map_col -c 1 -o gpurun_out/r02_k3_col -f python tests/ab_map.py > gpurun_out/r02_k3b.log 2>&1
LBG_MAP_COL=0 AB_MAPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:map_warp -c 1 -o gpurun_out/r02_k3_warp -f python tests/ab_map.py >> gpurun_out/r02_k3b.log 2>&1
