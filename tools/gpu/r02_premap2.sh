cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest -x -q tests/test_dropin.py > gpurun_out/r02_premap2_pytest.log 2>&1
PROBE_BLOCKS=2,2,2 PROBE_STEPS=4 timeout 600 python tests/coupled_probe.py scratch > /dev/null 2>&1
for pm in 0 1 0 1 0 1 0 1; do
  echo "PREMAP=$pm 2x2x2" >> gpurun_out/r02_premap2_probe.log
  LBDEM_GPU_PREMAP=$pm PROBE_BLOCKS=2,2,2 PROBE_STEPS=6 timeout 600 python tests/coupled_probe.py scratch >> gpurun_out/r02_premap2_probe.log 2>&1
done
for pm in 0 1; do
  echo "PREMAP=$pm 1 block" >> gpurun_out/r02_premap2_probe.log
  LBDEM_GPU_PREMAP=$pm PROBE_STEPS=5 timeout 600 python tests/coupled_probe.py scratch >> gpurun_out/r02_premap2_probe.log 2>&1
done
