cd $GRAFT_REPO_ROOT
for i in 1 2; do
  AB_STEPS=30 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_minb.log 2>&1
  LBG_LIB=$PWD/paper_2303_11811_b200/build_ab/liblbg.so AB_STEPS=30 timeout 300 python tests/ab_coupled_sweep.py | sed 's/{"env": {/{"env": {"MINB": "4", /' >> gpurun_out/r02_minb.log 2>&1
done
timeout 400 python tests/ab_config5_sweep.py >> gpurun_out/r02_minb.log 2>&1
LBG_LIB=$PWD/paper_2303_11811_b200/build_ab/liblbg.so timeout 400 python tests/ab_config5_sweep.py | sed 's/{"env": {/{"env": {"MINB": "4", /' >> gpurun_out/r02_minb.log 2>&1
