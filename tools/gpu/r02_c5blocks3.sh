cd $GRAFT_REPO_ROOT
for b in 16 8 16; do
  timeout 900 python bench_config5.py --gpus 1 --mode strong --force scratch --blocks-per-gpu $b --steps 3 >> gpurun_out/r02_c5blocks3_strong.log 2>&1
done
AB_REF=0 AB_BLOCKS="2,2,4:16;2,2,2:8;2,2,4:16;2,2,2:8" timeout 1700 python tests/ab_blocks.py >> gpurun_out/r02_c5blocks3_c3.log 2>&1
