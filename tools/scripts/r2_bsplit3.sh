cd $GRAFT_REPO_ROOT
python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 900 python -m pytest tests/test_gpu_step.py -q -p no:cacheprovider > gpurun_out/r2_bsplit3_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_bsplit3_tests.txt
echo done
