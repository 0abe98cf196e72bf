cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -m gpu -q -x > gpurun_out/r02_g27_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_g27_pytest.log
for env in "LBG_WALK_ROWS=1" "LBG_WALK_ROWS=0" "LBG_WALK_ROWS=1" "LBG_WALK_ROWS=0"; do
env $env AB_REDUCE=1 AB_STEPS=5 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_g27_ab.log 2>&1
done
AB_REDUCE=1 AB_STEPS=3 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g27_launches.csv python tests/ab_coupled_sweep.py > /dev/null 2>&1
