cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
  echo "process $i" >> gpurun_out/r02_sims_probe.log
  PROBE_SIMS=4 PROBE_BLOCKS=2,2,2 PROBE_STEPS=4 timeout 900 python tests/coupled_probe.py scratch 2>&1 | grep '"step": [23]' >> gpurun_out/r02_sims_probe.log
done
