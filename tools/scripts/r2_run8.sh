cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_t9_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_t9_tests.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_v3_bench.json 2> gpurun_out/r2_v3_bench.err
timeout 300 python bench.py --config tiny --steps 50 --warmup 5 > gpurun_out/r2_tiny.json 2> gpurun_out/r2_tiny.err
timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 > gpurun_out/r2_pmb.json 2> gpurun_out/r2_pmb.err
echo done
