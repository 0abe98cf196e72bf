# streamed host job on 2 GPUs: single-GPU job tests, multi-GPU job tests, config-4 bench at N = 2
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_job.py -q -x > gpurun_out/r02_job2_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_job2_pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "streamed_job or slab" > gpurun_out/r02_job2_multi.log 2>&1; echo rc=$? >> gpurun_out/r02_job2_multi.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02_job2_bench_n2.log 2>&1; echo rc=$? >> gpurun_out/r02_job2_bench_n2.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-coupled > gpurun_out/r02_job2_bench_n1.log 2>&1; echo rc=$? >> gpurun_out/r02_job2_bench_n1.log
