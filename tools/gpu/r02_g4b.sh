# 4 GPUs at HEAD: multi-GPU tests, config 5 weak and strong, config 4 (torchrun) with both halos
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests/test_gpu_multi.py tests/test_gpu_checked.py -m gpu -q -x > gpurun_out/r02_g4b_multi.log 2>&1; echo rc=$? >> gpurun_out/r02_g4b_multi.log
for n in 1 2 4; do
  timeout 1500 python bench_config5.py --gpus $n --steps 3 > gpurun_out/r02_g4b_c5_weak_n$n.log 2>&1; echo rc=$? >> gpurun_out/r02_g4b_c5_weak_n$n.log
done
for n in 1 2 4; do
  timeout 2400 python bench_config5.py --gpus $n --steps 3 --mode strong --force scratch > gpurun_out/r02_g4b_c5_strong_n$n.log 2>&1; echo rc=$? >> gpurun_out/r02_g4b_c5_strong_n$n.log
done
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r02_g4b_bench_n$n.log 2>&1; echo rc=$? >> gpurun_out/r02_g4b_bench_n$n.log
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus $n --steps 20 --warmup 5 --halo nccl --no-cpu-baseline > gpurun_out/r02_g4b_bench_nccl_n$n.log 2>&1; echo rc=$? >> gpurun_out/r02_g4b_bench_nccl_n$n.log
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29613 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02_g4b_ref_n4.log 2>&1; echo rc=$? >> gpurun_out/r02_g4b_ref_n4.log
