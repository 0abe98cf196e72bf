set -x
free -g; nproc; lscpu | grep -i "model name"
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_ref_arm.log 2>&1; echo rc=$? >> gpurun_out/r02_ref_arm.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench1.log 2>&1; echo rc=$? >> gpurun_out/r02_bench1.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r02_memcheck_parity.log 2>&1; echo rc=$? >> gpurun_out/r02_memcheck_parity.log
tail -3 gpurun_out/*.log
