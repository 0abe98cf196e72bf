cd $GRAFT_REPO_ROOT
lscpu -e > gpurun_out/r02_pin_lscpu.txt 2>&1; cat /sys/devices/system/cpu/cpu0/topology/thread_siblings_list >> gpurun_out/r02_pin_lscpu.txt 2>&1
PROBE_BLOCKS=2,2,2 PROBE_STEPS=4 timeout 600 python tests/coupled_probe.py scratch > /dev/null 2>&1
for i in 1 2 3 4; do
for v in "LBDEM_GPU_PIN_STRIDE=0" "LBDEM_GPU_PIN_STRIDE=1" "LBDEM_GPU_PIN_STRIDE=2"; do
  echo "$v" >> gpurun_out/r02_pin_probe.log
  env $v PROBE_BLOCKS=2,2,2 PROBE_STEPS=5 timeout 600 python tests/coupled_probe.py scratch 2>&1 | tail -2 >> gpurun_out/r02_pin_probe.log
done
done
