cd $GRAFT_REPO_ROOT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02_job3_bench_n2.log 2>&1; echo rc=$? >> gpurun_out/r02_job3_bench_n2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 20 --warmup 5 --halo nccl > gpurun_out/r02_job3_bench_n2_nccl.log 2>&1; echo rc=$? >> gpurun_out/r02_job3_bench_n2_nccl.log
nvidia-smi topo -m > gpurun_out/r02_job3_topo.txt 2>&1
