cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_graph.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x > gpurun_out/r2_t7_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_t7_tests.txt
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
for v in 0 4; do PPO_EXP_BWD_EPI=$v timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 > gpurun_out/r2_pmb_pf$v.json 2>&1; done
timeout 1200 python tools/ab_variants.py --B 38400 --var PPO_EXP_BWD_EPI --vals 0,4 --rounds 3 --steps 3 > gpurun_out/r2_ab_bwd_prefetch.txt 2>&1
timeout 1200 python tools/ab_variants.py --B 38400 --var PPO_VARIANT_FWD --vals pair,pair2 --rounds 3 --steps 3 > gpurun_out/r2_ab_fwd_pair2.txt 2>&1
echo done
