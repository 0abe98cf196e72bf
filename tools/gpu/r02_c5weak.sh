cd $GRAFT_REPO_ROOT
for b in 4 8 16 4 8 16; do
  timeout 900 python bench_config5.py --gpus 1 --mode weak --force scratch --blocks-per-gpu $b --steps 3 >> gpurun_out/r02_c5weak_ab.log 2>&1
done
