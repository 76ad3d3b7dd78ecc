cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 PPO_NVCC_EXTRA="-DPPO_TRACE" python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
for v in 0 1 2 3; do
echo "== PPO_EXP_BWD_EPI=$v" >> gpurun_out/r2_trace_bwd_exp.txt
PPO_EXP_BWD_EPI=$v PPO_VARIANT_WGRAD=1cta PPO_VARIANT_WGRAD_O=1cta timeout 300 python tools/trace_step.py --bwd --B 600 --H 4096 --D 4032 --mhz 1800 2>&1 | head -4 | cut -c1-400 >> gpurun_out/r2_trace_bwd_exp.txt
done
python paper_1912_06680_b200/build.py > /dev/null 2>&1
echo done
