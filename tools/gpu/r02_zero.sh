# map_zero_kernel A/B (mapping wall time + fraction hash) and the mapping/drop-in parity tests
cd $GRAFT_REPO_ROOT
P=paper_2303_11811_b200
for rep in 1 2; do
  for v in "" build_oldzero; do
    lib=$P/liblbg.so; [ -n "$v" ] && lib=$P/$v/liblbg.so
    echo "lib=$v" >> gpurun_out/r02_zero_ab.log
    LBG_LIB=$lib AB_MAPS=20 timeout 300 python tests/ab_map.py >> gpurun_out/r02_zero_ab.log 2>&1
  done
done
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py tests/test_gpu_fullsize.py tests/test_gpu_job.py -q -x > gpurun_out/r02_zero_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_zero_pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:map_zero -c 6 --csv python tests/ab_map.py > gpurun_out/r02_zero_ncu.csv 2>&1
