cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,power.draw --format=csv > gpurun_out/r2_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r2_t1_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_t1_tests.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_t1_bench.json 2> gpurun_out/r2_t1_bench.err
echo "bench rc=$?"
