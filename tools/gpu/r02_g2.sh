# K12 unified coupled sweep: parity subset + A/B on config 3's bed
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -m gpu -q -x -k "coupled or setu or fused or mapping_and_solid or shear or sweep or config1_known_answers or particle_bed or decomposition_invariance" > gpurun_out/r02_g2_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02_g2_pytest.log
for env in "LBG_K12=0" "LBG_K12=1" "LBG_K12_SM=4" "LBG_K12_SM=6" "LBG_K12_PF=0" "LBG_K12_PF=0 LBG_K12_SM=4" "LBG_K12=1"; do
  env $env timeout 300 python tests/ab_coupled_sweep.py >> gpurun_out/r02_g2_ab.log 2>&1
done
