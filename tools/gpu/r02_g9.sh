cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py tests/test_gpu_reference_cases.py -m gpu -q -x > gpurun_out/r02_g9_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_g9_pytest.log
AB_REDUCE=1 AB_STEPS=30 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_g9_ab.log 2>&1
PROBE_STEPS=3 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g9_launches.csv python tests/coupled_probe.py scratch > /dev/null 2>&1
timeout 2400 python -m pytest tests/test_gpu_variants.py -m gpu -q -x > gpurun_out/r02_g9_variants.log 2>&1; echo rc=$? >> gpurun_out/r02_g9_variants.log
