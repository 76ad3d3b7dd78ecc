cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 900 python -m pytest tests/test_gpu_kernels.py -k "gae" -q -p no:cacheprovider > gpurun_out/r2_gae_fast3_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_gae_fast3_tests.txt
rm -f gpurun_out/r2_gae_fast3.txt
for r in 1 2; do timeout 300 python tools/gae_probe.py --L 256,1350,6300,20000,100000,1000000 --steps 1000000000 >> gpurun_out/r2_gae_fast3.txt 2>&1; done
echo done
