cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_aa.py -m gpu -q -x > gpurun_out/r02_g10_aa.log 2>&1; echo rc=$? >> gpurun_out/r02_g10_aa.log
timeout 3000 python -m pytest tests/test_gpu_checked.py -m gpu -q -x > gpurun_out/r02_g10_checked.log 2>&1; echo rc=$? >> gpurun_out/r02_g10_checked.log
AB_STEPS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_chain -s 3 -c 1 -o gpurun_out/r02_walk python tests/ab_coupled_sweep.py > /dev/null 2>&1
AB_REDUCE=1 AB_STEPS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:walk_chain -s 1 -c 1 -o gpurun_out/r02_walk python tests/ab_coupled_sweep.py > gpurun_out/r02_g10_ncu.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02_g10_bench.log 2>&1; echo rc=$? >> gpurun_out/r02_g10_bench.log
