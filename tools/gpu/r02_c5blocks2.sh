cd $GRAFT_REPO_ROOT
for b in 16 8 16; do
  timeout 900 python bench_config5.py --gpus 1 --mode strong --force scratch --blocks-per-gpu $b --steps 3 >> gpurun_out/r02_c5blocks2_strong.log 2>&1
done
