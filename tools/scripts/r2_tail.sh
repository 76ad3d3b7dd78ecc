cd $GRAFT_REPO_ROOT
python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_tail_gpu_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_tail_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_tail_smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/r2_tail_smoke.txt
timeout 300 python bench.py --config tiny --steps 200 --warmup 20 > gpurun_out/r2_tail_tiny.json 2> /dev/null
timeout 900 python bench.py > gpurun_out/r2_tail_bench.json 2> /dev/null
timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 > gpurun_out/r2_tail_pmb.json 2> /dev/null
echo done
