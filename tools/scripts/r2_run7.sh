cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_graph.py -q -p no:cacheprovider -x > gpurun_out/r2_t8_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_t8_tests.txt
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
rm -f gpurun_out/r2_gae_var2.txt
for v in 0 3 6 7 8; do echo "variant $v" >> gpurun_out/r2_gae_var2.txt; PPO_GAE_VARIANT=$v timeout 300 python tools/gae_probe.py --L 1350,20000,100000,1000000 --steps 1000000000 >> gpurun_out/r2_gae_var2.txt 2>&1; done
timeout 1200 python tools/ab_variants.py --B 38400 --var PPO_EXP_BWD_EPI --vals 0,8 --rounds 3 --steps 3 > gpurun_out/r2_ab_bwd_ahead.txt 2>&1
for v in 0 8; do PPO_EXP_BWD_EPI=$v timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 > gpurun_out/r2_pmb_ahead$v.json 2>&1; done
echo done
