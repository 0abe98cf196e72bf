cd $GRAFT_REPO_ROOT
timeout 1200 python bench_config5.py --gpus 1 --mode strong --force scratch --steps 3 > gpurun_out/r02_c5strong2_n1_b16.log 2>&1
timeout 1200 python bench_config5.py --gpus 4 --mode strong --force scratch --steps 3 --blocks-per-gpu 4 > gpurun_out/r02_c5strong2_n4_b4.log 2>&1
timeout 1200 python bench_config5.py --gpus 4 --mode strong --force scratch --steps 3 --blocks-per-gpu 8 > gpurun_out/r02_c5strong2_n4_b8.log 2>&1
timeout 1200 python bench_config5.py --gpus 2 --mode strong --force scratch --steps 3 --blocks-per-gpu 8 > gpurun_out/r02_c5strong2_n2_b8.log 2>&1
timeout 1200 python bench_config5.py --gpus 4 --mode strong --force scratch --steps 3 --blocks-per-gpu 4 > gpurun_out/r02_c5strong2_n4_b4b.log 2>&1
