# 4-GPU box at HEAD: multi-GPU suite, config 4 bench at N = 2 and 4 (streamed-job e2e), reference arm under torchrun
cd $GRAFT_REPO_ROOT
nvidia-smi topo -m > gpurun_out/r02_four_topo.txt 2>&1
timeout 2400 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/r02_four_multi.log 2>&1; echo rc=$? >> gpurun_out/r02_four_multi.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02_four_bench_n4.log 2>&1; echo rc=$? >> gpurun_out/r02_four_bench_n4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29622 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02_four_bench_n2.log 2>&1; echo rc=$? >> gpurun_out/r02_four_bench_n2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29623 bench.py --gpus 4 --steps 20 --warmup 5 --halo nccl > gpurun_out/r02_four_bench_n4_nccl.log 2>&1; echo rc=$? >> gpurun_out/r02_four_bench_n4_nccl.log
