cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_job.py -q -x > gpurun_out/r02_job4_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_job4_pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "streamed_job" > gpurun_out/r02_job4_multi.log 2>&1; echo rc=$? >> gpurun_out/r02_job4_multi.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-coupled > gpurun_out/r02_job4_bench_n1.log 2>&1; echo rc=$? >> gpurun_out/r02_job4_bench_n1.log
