cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py tests/test_gpu_reference_cases.py tests/test_abi.py -m gpu -q -x -s > gpurun_out/r02_g8_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_g8_pytest.log
AB_REDUCE=1 AB_STEPS=30 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_g8_ab.log 2>&1
PROBE_STEPS=5 timeout 600 python tests/coupled_probe.py scratch > gpurun_out/r02_g8_probe1.log 2>&1
LBDEM_GPU_PREMAP=0 PROBE_STEPS=5 timeout 600 python tests/coupled_probe.py scratch > gpurun_out/r02_g8_probe1_nopremap.log 2>&1
PROBE_BLOCKS=2,2,2 PROBE_STEPS=5 timeout 600 python tests/coupled_probe.py scratch > gpurun_out/r02_g8_probe8.log 2>&1
LBDEM_GPU_PREMAP=0 PROBE_BLOCKS=2,2,2 PROBE_STEPS=5 timeout 600 python tests/coupled_probe.py scratch > gpurun_out/r02_g8_probe8_nopremap.log 2>&1
PROBE_STEPS=3 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g8_launches.csv python tests/coupled_probe.py scratch > /dev/null 2>&1
