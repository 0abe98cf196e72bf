cd $GRAFT_REPO_ROOT
for env in "LBG_MAP_COL=2" "LBG_MAP_COL=2 LBG_MAP_CTA_WARPS=4" "LBG_MAP_COL=3" "LBG_MAP_COL=3 LBG_MAP_CTA_WARPS=4"; do
  env $env timeout 300 python tests/ab_map.py >> gpurun_out/r02_k3e_ab.log 2>&1
  env $env AB_MAPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"map_|bin_" --csv \
     --log-file gpurun_out/r02_k3e_$(echo $env | tr ' =' '__').csv python tests/ab_map.py > /dev/null 2>&1
done
LBG_MAP_COL=3 timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_reference_cases.py > gpurun_out/r02_k3e_pytest.log 2>&1
