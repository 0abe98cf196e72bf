cd $GRAFT_REPO_ROOT
P=paper_2303_11811_b200
for rep in 1 2; do
for v in "" build_minb4; do
  lib=$P/liblbg.so; [ -n "$v" ] && lib=$P/$v/liblbg.so
  echo "lib=$v" >> gpurun_out/r02_minb_ab3.log
  LBG_LIB=$lib AB_STEPS=30 timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_minb_ab3.log 2>&1
done
done
