cd $GRAFT_REPO_ROOT
LBG_WALK_ONE_BELOW=100000000 timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -q -x > gpurun_out/r02_walk1_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_walk1_pytest.log
for rep in 1 2; do
for v in 0 100000000; do
  LBG_WALK_ONE_BELOW=$v LBG_REDUCE_PROFILE=0 AB_REDUCE=1 AB_STEPS=10 timeout 600 python tests/ab_coupled_sweep.py >> gpurun_out/r02_walk1_reduce.log 2>&1
  LBG_WALK_ONE_BELOW=$v AB_REF=0 AB_BLOCKS="2,2,4:16" timeout 900 python tests/ab_blocks.py >> gpurun_out/r02_walk1_c3.log 2>&1
done
done
