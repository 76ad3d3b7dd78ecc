cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > gpurun_out/r2_mca_build.txt 2>&1 || echo build failed
PPO_VARIANT_WGRAD=pairmc timeout 900 python -m pytest tests/test_gpu_step.py -x -q -p no:cacheprovider > gpurun_out/r2_mca_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_mca_tests.txt
timeout 1200 python tools/ab_variants.py --B 38400 --steps 3 --rounds 3 --var PPO_VARIANT_WGRAD --vals pair,pairmc > gpurun_out/r2_mca_ab.txt 2>&1
echo "ab rc=$?" >> gpurun_out/r2_mca_ab.txt
rm -f gpurun_out/r2_gae_var7.txt
for v in 0 7 9 10; do echo "variant $v" >> gpurun_out/r2_gae_var7.txt; PPO_GAE_VARIANT=$v timeout 300 python tools/gae_probe.py --L 1350,6300,20000,1000000 --steps 1000000000 >> gpurun_out/r2_gae_var7.txt 2>&1; done
echo done
