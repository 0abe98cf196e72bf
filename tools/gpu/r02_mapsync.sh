cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest -x -q tests/test_dropin.py > gpurun_out/r02_mapsync_pytest.log 2>&1
PROBE_BLOCKS=2,2,2 PROBE_STEPS=4 timeout 600 python tests/coupled_probe.py scratch > /dev/null 2>&1
for i in 1 2 3 4; do
  echo "run $i 2x2x2" >> gpurun_out/r02_mapsync_probe.log
  PROBE_BLOCKS=2,2,2 PROBE_STEPS=6 timeout 600 python tests/coupled_probe.py scratch >> gpurun_out/r02_mapsync_probe.log 2>&1
done
echo "1 block" >> gpurun_out/r02_mapsync_probe.log
PROBE_STEPS=5 timeout 600 python tests/coupled_probe.py scratch >> gpurun_out/r02_mapsync_probe.log 2>&1
