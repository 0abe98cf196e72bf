# 4 GPUs: multi-GPU tests, config 4 (torchrun) and config 5 weak scaling through the drop-in
cd $GRAFT_REPO_ROOT
nvidia-smi topo -m > gpurun_out/r02_g12_topo.txt 2>&1
timeout 2400 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -s > gpurun_out/r02_g12_multi.log 2>&1; echo rc=$? >> gpurun_out/r02_g12_multi.log
for n in 1 2 4; do
  timeout 1500 python bench_config5.py --gpus $n --steps 3 > gpurun_out/r02_g12_c5_n$n.log 2>&1; echo rc=$? >> gpurun_out/r02_g12_c5_n$n.log
done
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/r02_g12_bench_n$n.log 2>&1; echo rc=$? >> gpurun_out/r02_g12_bench_n$n.log
done
