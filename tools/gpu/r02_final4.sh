# 4-GPU box at the end of round 2: multi-GPU suite, config 4 bench at N = 2 and 4, reference arm under torchrun
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/r02_end4_multi.log 2>&1; echo rc=$? >> gpurun_out/r02_end4_multi.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02_end4_bench_n2.log 2>&1; echo rc=$? >> gpurun_out/r02_end4_bench_n2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02_end4_bench_n4.log 2>&1; echo rc=$? >> gpurun_out/r02_end4_bench_n4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29633 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02_end4_ref_n4.log 2>&1; echo rc=$? >> gpurun_out/r02_end4_ref_n4.log
