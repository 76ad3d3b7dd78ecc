cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 1500 python tools/ab_variants.py --B 38400 --var PPO_MULTISTEP --vals 1,2 --rounds 3 --steps 3 > gpurun_out/r2_ab_multistep_big.txt 2>&1
echo done
