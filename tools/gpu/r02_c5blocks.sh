# config 5 on 1 GPU: host parallelism (x-slab blocks per GPU = host workers) A/B, scratch mode
cd $GRAFT_REPO_ROOT
for b in 4 8 15; do
  timeout 900 python bench_config5.py --gpus 1 --mode strong --force scratch --blocks-per-gpu $b --steps 3 >> gpurun_out/r02_c5blocks_strong.log 2>&1
done
for b in 4 8 15; do
  timeout 600 python bench_config5.py --gpus 1 --mode weak --force scratch --blocks-per-gpu $b --steps 3 >> gpurun_out/r02_c5blocks_weak.log 2>&1
done
