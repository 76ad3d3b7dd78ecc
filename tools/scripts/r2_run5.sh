cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2_t5_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_t5_tests.txt
timeout 300 python bench.py --config tiny --steps 50 --warmup 5 > gpurun_out/r2_tiny.json 2> gpurun_out/r2_tiny.err
timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 > gpurun_out/r2_pmb.json 2> gpurun_out/r2_pmb.err
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_v2_bench.json 2> gpurun_out/r2_v2_bench.err
PPO_EXPERIMENTS=1 PPO_NVCC_EXTRA="-DPPO_TRACE" python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
PPO_VARIANT_HEADS=1cta timeout 300 python tools/trace_step.py --B 32 --H 128 --D 256 > gpurun_out/r2_trace3.txt 2>&1
PPO_VARIANT_HEADS=1cta timeout 300 python tools/trace_step.py --B 600 --H 4096 --D 4032 --mhz 1800 >> gpurun_out/r2_trace3.txt 2>&1
echo done
