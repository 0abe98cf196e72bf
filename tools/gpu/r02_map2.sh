cd $GRAFT_REPO_ROOT
P=paper_2303_11811_b200
for rep in 1 2; do
for v in "" build_oldmap; do
  lib=$P/liblbg.so; [ -n "$v" ] && lib=$P/$v/liblbg.so
  LBG_LIB=$lib AB_MAPS=6 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:map_col_kernel --csv python tests/ab_map.py > gpurun_out/r02_map2_${rep}_${v:-new}.csv 2>&1
done
done
