cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_job.py -q -x > gpurun_out/r02_tail_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_tail_pytest.log
for rep in 1 2 3; do
for t in 0 4 16; do
  echo "tail=$t" >> gpurun_out/r02_tail_ab.log
  LBG_JOB_TAIL=$t AB_SLABS=16 timeout 600 python tests/ab_job.py 512 20 2>&1 | grep slab >> gpurun_out/r02_tail_ab.log
done
done
