cd $GRAFT_REPO_ROOT
AB_STEPS=3 timeout 900 ncu --set full --import-source on --clock-control none -k regex:unified -s 3 -c 1 -o gpurun_out/r02_unified python tests/ab_coupled_sweep.py > gpurun_out/r02_g4_ncu.log 2>&1
echo rc=$? >> gpurun_out/r02_g4_ncu.log
