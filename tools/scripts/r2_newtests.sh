cd $GRAFT_REPO_ROOT
python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 1500 python -m pytest tests/test_gpu_graph.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > gpurun_out/r2_newtests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_newtests.txt
echo done
