# K12: prefetch flavours + ncu of the unified kernel on config 3's bed
cd $GRAFT_REPO_ROOT
for env in "LBG_K12_PF=0" "LBG_K12_PF=2" "LBG_K12_PF=2 LBG_K12_SM=4" "LBG_K12=0" "LBG_K12_PF=0"; do
  env $env AB_STEPS=30 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_g3_ab.log 2>&1
done
AB_STEPS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:coupled_unified -s 6 -c 1 -o gpurun_out/r02_unified python tests/ab_coupled_sweep.py > gpurun_out/r02_g3_ncu.log 2>&1
echo rc=$? >> gpurun_out/r02_g3_ncu.log
