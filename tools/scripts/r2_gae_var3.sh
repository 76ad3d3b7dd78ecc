cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
rm -f gpurun_out/r2_gae_var3.txt
for v in 0 9 10 1 2; do echo "variant $v" >> gpurun_out/r2_gae_var3.txt; PPO_GAE_VARIANT=$v timeout 300 python tools/gae_probe.py --L 256,1350,6300,20000 --steps 1000000000 >> gpurun_out/r2_gae_var3.txt 2>&1; done
python paper_1912_06680_b200/build.py > /dev/null 2>&1
echo done
