# streamed host job: parity tests + bench e2e
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_job.py -q -x > gpurun_out/r02_job1_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_job1_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-coupled > gpurun_out/r02_job1_bench.log 2>&1; echo rc=$? >> gpurun_out/r02_job1_bench.log
