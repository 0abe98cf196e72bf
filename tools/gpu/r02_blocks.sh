cd $GRAFT_REPO_ROOT
PROBE_BLOCKS=2,2,2 PROBE_STEPS=4 timeout 600 python tests/coupled_probe.py scratch > /dev/null 2>&1
for b in "2,2,2 8" "4,2,2 16" "2,2,4 16" "2,2,2 8" "4,2,2 16" "2,2,4 16" "4,4,1 16" "2,4,2 16"; do
  set -- $b
  echo "blocks $1 workers $2" >> gpurun_out/r02_blocks_probe.log
  PROBE_BLOCKS=$1 PROBE_WORKERS=$2 PROBE_STEPS=6 timeout 600 python tests/coupled_probe.py scratch >> gpurun_out/r02_blocks_probe.log 2>&1
done
