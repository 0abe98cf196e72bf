# config 5 weak with the default host parallelism (8 x-slab blocks per GPU within the CPUs), 1 / 2 / 4 GPUs, both force modes
cd $GRAFT_REPO_ROOT
for g in 1 2 4; do
  timeout 900 python bench_config5.py --gpus $g --mode weak --force both --steps 3 > gpurun_out/r02_c5weak4_n$g.log 2>&1
done
timeout 900 python bench_config5.py --gpus 4 --mode weak --force scratch --steps 3 > gpurun_out/r02_c5weak4_n4b.log 2>&1
