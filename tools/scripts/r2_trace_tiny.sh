cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 PPO_NVCC_EXTRA="-DPPO_TRACE -DPPO_TRACE_UNIT=8" python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
rm -f gpurun_out/r2_trace_tiny.txt
echo "== forward (multi-step), unit 8 = step 8" >> gpurun_out/r2_trace_tiny.txt
PPO_VARIANT_HEADS=1cta timeout 300 python tools/trace_step.py --B 32 --H 128 --D 256 --mhz 1965 >> gpurun_out/r2_trace_tiny.txt 2>&1
echo "== backward (multi-step), unit 8 = step 8 (time 7)" >> gpurun_out/r2_trace_tiny.txt
PPO_VARIANT_HEADS=1cta PPO_VARIANT_WGRAD=1cta PPO_VARIANT_WGRAD_O=1cta timeout 300 python tools/trace_step.py --bwd --B 32 --H 128 --D 256 --mhz 1965 >> gpurun_out/r2_trace_tiny.txt 2>&1
python paper_1912_06680_b200/build.py > /dev/null 2>&1
echo done
