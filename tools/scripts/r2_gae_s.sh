cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
rm -f gpurun_out/r2_gae_var7.txt
for v in 0 7 9 10; do echo "variant $v" >> gpurun_out/r2_gae_var7.txt; PPO_GAE_VARIANT=$v timeout 300 python tools/gae_probe.py --L 1350,6300,20000,1000000 --steps 1000000000 >> gpurun_out/r2_gae_var7.txt 2>&1; done
python paper_1912_06680_b200/build.py > /dev/null 2>&1
echo done
