# config 5 on the 4-GPU box at HEAD: strong (host workers = CPUs) and weak (4 blocks per GPU), scratch (bitwise) mode
cd $GRAFT_REPO_ROOT
nproc > gpurun_out/r02_c5scale_nproc.txt
for g in 1 2 4; do
  timeout 1200 python bench_config5.py --gpus $g --mode strong --force scratch --steps 3 > gpurun_out/r02_c5scale_strong_n$g.log 2>&1
done
for g in 1 2 4; do
  timeout 900 python bench_config5.py --gpus $g --mode weak --force both --steps 3 > gpurun_out/r02_c5scale_weak_n$g.log 2>&1
done
