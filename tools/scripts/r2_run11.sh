cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_t11_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_t11_tests.txt
timeout 600 python bench.py --config gae --steps 5 --warmup 2 > gpurun_out/r2_gae_bench.json 2> gpurun_out/r2_gae_bench.err
timeout 300 python bench.py --config tiny --steps 50 --warmup 5 > gpurun_out/r2_tiny.json 2> gpurun_out/r2_tiny.err
echo done
