cd $GRAFT_REPO_ROOT
python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_bsplit2_gpu_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_bsplit2_gpu_tests.txt
timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 > gpurun_out/r2_bsplit2_pmb.json 2> gpurun_out/r2_bsplit2_pmb.err
timeout 300 python bench.py --config tiny --steps 50 --warmup 5 > gpurun_out/r2_bsplit2_tiny.json 2> gpurun_out/r2_bsplit2_tiny.err
echo done
