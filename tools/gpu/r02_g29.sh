cd $GRAFT_REPO_ROOT
start=$(date +%s)
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_g29_bench.log 2> gpurun_out/r02_g29_bench.err; echo rc=$? >> gpurun_out/r02_g29_bench.log
echo "wall_s=$(( $(date +%s) - start ))" >> gpurun_out/r02_g29_bench.log
