cd $GRAFT_REPO_ROOT
bash tools/scripts/r2_ncu_cublas.sh
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 900 python tools/ab_variants.py --B 38400 --var PPO_EXP_BWD_EPI --vals 0,1,2,3 --rounds 2 --steps 3 > gpurun_out/r2_ab_bwd_epi.txt 2>&1
echo ab done
