cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest -x -q tests/test_dropin.py > gpurun_out/r02_spin_pytest.log 2>&1
LBDEM_GPU_SPIN_PHASES=0 timeout 1200 python -m pytest -x -q tests/test_dropin.py -k "bed or decomposition or overfull" >> gpurun_out/r02_spin_pytest.log 2>&1
PROBE_BLOCKS=2,2,2 PROBE_STEPS=4 timeout 600 python tests/coupled_probe.py scratch > /dev/null 2>&1
for sp in 0 1 0 1 0 1; do
  echo "SPIN=$sp 2x2x2" >> gpurun_out/r02_spin_probe.log
  LBDEM_GPU_SPIN_PHASES=$sp PROBE_BLOCKS=2,2,2 PROBE_STEPS=6 timeout 600 python tests/coupled_probe.py scratch >> gpurun_out/r02_spin_probe.log 2>&1
done
