# validation at HEAD: full GPU suite, smoke, bench (N = 1), reference arm
cd $GRAFT_REPO_ROOT
timeout 5400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_head2_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_head2_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_head2_smoke.log 2>&1; echo rc=$? >> gpurun_out/r02_head2_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_head2_bench.log 2>&1; echo rc=$? >> gpurun_out/r02_head2_bench.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_head2_ref.log 2>&1; echo rc=$? >> gpurun_out/r02_head2_ref.log
