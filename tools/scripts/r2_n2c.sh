cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_dp_multi.py -q -p no:cacheprovider > gpurun_out/r2_n2_tests2.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_n2_tests2.txt
echo done
