cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 1200 python tools/ab_variants.py --B 38400 --var PPO_EXP_BWD_EPI --vals 0,8 --rounds 3 --steps 3 > gpurun_out/r2_ab_bwd_ahead.txt 2>&1
for v in 0 8; do PPO_EXP_BWD_EPI=$v timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 > gpurun_out/r2_pmb_ahead$v.json 2>&1; done
echo done
