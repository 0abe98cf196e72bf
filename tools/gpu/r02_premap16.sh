cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  for pm in 0 1; do
    echo "premap=$pm" >> gpurun_out/r02_premap16.log
    LBDEM_GPU_PREMAP=$pm AB_REF=0 AB_BLOCKS="2,2,4:16" timeout 900 python tests/ab_blocks.py >> gpurun_out/r02_premap16.log 2>&1
  done
done
