cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -m gpu -q -x > gpurun_out/r02_g22_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_g22_pytest.log
AB_REDUCE=1 AB_STEPS=10 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_g22_ab.log 2>&1
AB_REDUCE=1 AB_STEPS=3 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g22_launches.csv python tests/ab_coupled_sweep.py > /dev/null 2>&1
PROBE_STEPS=5 timeout 600 python tests/coupled_probe.py scratch > gpurun_out/r02_g22_probe1.log 2>&1
PROBE_BLOCKS=2,2,2 PROBE_STEPS=5 timeout 600 python tests/coupled_probe.py scratch > gpurun_out/r02_g22_probe8.log 2>&1
