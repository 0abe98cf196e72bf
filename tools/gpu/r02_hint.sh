# A/B: cache hints on the coupled sweep's PDF loads/stores (config 3 bed and config 5 block)
cd $GRAFT_REPO_ROOT
P=paper_2303_11811_b200
for rep in 1 2; do
for v in "" build_stcs build_ldcs build_ldna; do
  lib=$P/liblbg.so; [ -n "$v" ] && lib=$P/$v/liblbg.so
  echo "lib=$v" >> gpurun_out/r02_hint_ab3.log
  LBG_LIB=$lib AB_STEPS=30 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_hint_ab3.log 2>&1
done
done
for v in "" build_stcs; do
  lib=$P/liblbg.so; [ -n "$v" ] && lib=$P/$v/liblbg.so
  echo "lib=$v" >> gpurun_out/r02_hint_ab5.log
  LBG_LIB=$lib timeout 400 python tests/ab_config5_sweep.py >> gpurun_out/r02_hint_ab5.log 2>&1
done
