cd $GRAFT_REPO_ROOT
PROBE_BLOCKS=2,2,2 PROBE_STEPS=4 timeout 600 python tests/coupled_probe.py scratch > /dev/null 2>&1
for i in 1 2 3 4 5; do
for v in "LBDEM_GPU_SPIN_PHASES=0" "LBDEM_GPU_SPIN_US=2000" "LBDEM_GPU_SPIN_US=50"; do
  echo "$v" >> gpurun_out/r02_spin2_probe.log
  env $v PROBE_BLOCKS=2,2,2 PROBE_STEPS=5 timeout 600 python tests/coupled_probe.py scratch 2>&1 | tail -2 >> gpurun_out/r02_spin2_probe.log
done
done
