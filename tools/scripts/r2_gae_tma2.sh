cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
for v in 6 7; do PPO_GAE_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_kernels.py -k gae -q -p no:cacheprovider > gpurun_out/r2_gae_tma_tests$v.txt 2>&1; done
rm -f gpurun_out/r2_gae_var6.txt
for v in 0 6 7; do echo "variant $v" >> gpurun_out/r2_gae_var6.txt; PPO_GAE_VARIANT=$v timeout 300 python tools/gae_probe.py --L 256,1350,6300,20000,100000,1000000 --steps 1000000000 >> gpurun_out/r2_gae_var6.txt 2>&1; done
python paper_1912_06680_b200/build.py > /dev/null 2>&1
echo done
