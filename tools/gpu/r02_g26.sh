cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_aa.py -m gpu -q -x > gpurun_out/r02_g26_aa.log 2>&1; echo rc=$? >> gpurun_out/r02_g26_aa.log
for bx in 128 256 64 32 128; do
  LBG_AA_BX=$bx timeout 300 python tests/ab_config2_variants.py >> gpurun_out/r02_g26_ab.log 2>&1
done
