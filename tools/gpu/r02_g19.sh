cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_aa.py -m gpu -q -x > gpurun_out/r02_g19_aa.log 2>&1; echo rc=$? >> gpurun_out/r02_g19_aa.log
timeout 300 python tests/ab_config2_variants.py >> gpurun_out/r02_g19_ab.log 2>&1
timeout 300 python tests/ab_config2_variants.py >> gpurun_out/r02_g19_ab.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_g19_launches.csv python tests/ab_config2_variants.py > /dev/null 2>&1
