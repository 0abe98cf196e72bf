# ncu launch list of the bench command (kernel shares; serialised, cold-cache)
cd $GRAFT_REPO_ROOT
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02_launches2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_launches2_bench.log 2>&1; echo rc=$? >> gpurun_out/r02_launches2_bench.log
