cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 1200 python tools/ab_variants.py --B 38400 --var PPO_VARIANT_FWD --vals pair,pair2 --rounds 3 --steps 3 > gpurun_out/r2_ab_fwd_pair2.txt 2>&1
echo done
