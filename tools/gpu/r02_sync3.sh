cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest -x -q tests/test_dropin.py > gpurun_out/r02_sync4_pytest.log 2>&1
timeout 1200 python -m pytest -x -q tests/test_gpu_variants.py -k "FAST_SYNC" >> gpurun_out/r02_sync4_pytest.log 2>&1
PROBE_BLOCKS=2,2,2 PROBE_STEPS=4 timeout 600 python tests/coupled_probe.py scratch > /dev/null 2>&1
for fs in 0 1 0 1; do
  echo "FAST_SYNC=$fs 2x2x2" >> gpurun_out/r02_sync4_probe.log
  LBDEM_GPU_FAST_SYNC=$fs PROBE_BLOCKS=2,2,2 PROBE_STEPS=6 timeout 600 python tests/coupled_probe.py scratch >> gpurun_out/r02_sync4_probe.log 2>&1
done
for fs in 0 1; do
  echo "FAST_SYNC=$fs 1 block" >> gpurun_out/r02_sync4_probe.log
  LBDEM_GPU_FAST_SYNC=$fs PROBE_STEPS=5 timeout 600 python tests/coupled_probe.py scratch >> gpurun_out/r02_sync4_probe.log 2>&1
done
nproc > gpurun_out/r02_sync4_host.txt; lscpu | head -20 >> gpurun_out/r02_sync4_host.txt
