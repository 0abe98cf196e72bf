cd $GRAFT_REPO_ROOT
for env in "LBG_MAP_ILP=0" "LBG_MAP_ILP=1" "LBG_MAP_ILP=2"; do
  env $env timeout 300 python tests/ab_map.py >> gpurun_out/r02_k3f_ab.log 2>&1
  env $env AB_MAPS=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"map_" --csv \
     --log-file gpurun_out/r02_k3f_$(echo $env | tr ' =' '__').csv python tests/ab_map.py > /dev/null 2>&1
done
