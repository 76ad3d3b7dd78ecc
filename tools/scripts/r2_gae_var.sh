cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
for v in 0 1 2 3 4 5; do echo "variant $v" >> gpurun_out/r2_gae_var.txt; PPO_GAE_VARIANT=$v timeout 300 python tools/gae_probe.py --L 1350,6300,20000,100000,1000000 --steps 1000000000 >> gpurun_out/r2_gae_var.txt 2>&1; done
echo done
