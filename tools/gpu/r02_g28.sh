cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -m gpu -q -x > gpurun_out/r02_g28_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_g28_pytest.log
LBG_WALK_ROWS=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -m gpu -q -x -k "hydro or finalize or fused or bed or config or coupled" > gpurun_out/r02_g28_pytest_rows.log 2>&1; echo rc=$? >> gpurun_out/r02_g28_pytest_rows.log
