cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_graph.py tests/test_gpu_aux.py -q -p no:cacheprovider -x > gpurun_out/r2_t10_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_t10_tests.txt
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
for i in 1 2; do for v in 0 1; do PPO_BWD_NARROW=$v timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 > gpurun_out/r2_pmb_narrow$v.$i.json 2>&1; done; done
python paper_1912_06680_b200/build.py > /dev/null 2>&1
timeout 300 python bench.py --config tiny --steps 50 --warmup 5 > gpurun_out/r2_tiny.json 2> gpurun_out/r2_tiny.err
echo done
