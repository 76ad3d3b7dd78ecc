cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
for var in PPO_EXP_APOL_wgrad_xh PPO_EXP_BPOL_wgrad_xh PPO_EXP_APOL_lstm_fwd_step PPO_EXP_BPOL_lstm_fwd_step PPO_EXP_APOL_lstm_bwd_step PPO_EXP_BPOL_lstm_bwd_step; do
timeout 900 python tools/ab_variants.py --B 38400 --var $var --vals 0,1,2 --rounds 2 --steps 2 >> gpurun_out/r2_ab_pol.txt 2>&1
done
echo done
