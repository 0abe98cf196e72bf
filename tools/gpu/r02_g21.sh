cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -m gpu -q -x -k "map or coupled or bed or config or fullsize" > gpurun_out/r02_g21_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_g21_pytest.log
LBG_MAP_MINB=5 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "map" > gpurun_out/r02_g21_pytest5.log 2>&1; echo rc=$? >> gpurun_out/r02_g21_pytest5.log
AB_STEPS=3 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g21_launches4.csv python tests/ab_coupled_sweep.py > /dev/null 2>&1
LBG_MAP_MINB=5 AB_STEPS=3 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g21_launches5.csv python tests/ab_coupled_sweep.py > /dev/null 2>&1
