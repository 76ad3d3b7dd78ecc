cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 PPO_NVCC_EXTRA="-DPPO_TRACE" python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
PPO_VARIANT_WGRAD=1cta PPO_VARIANT_WGRAD_O=1cta timeout 300 python tools/trace_step.py --bwd --B 600 --H 4096 --D 4032 --mhz 1800 > gpurun_out/r2_trace_bwd.txt 2>&1
PPO_VARIANT_WGRAD=1cta PPO_VARIANT_WGRAD_O=1cta timeout 300 python tools/trace_step.py --bwd --B 32 --H 128 --D 256 >> gpurun_out/r2_trace_bwd.txt 2>&1
python paper_1912_06680_b200/build.py > /dev/null 2>&1
bash tools/scripts/r2_gae_ncu.sh
echo done
