cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
for i in 1 2; do for v in 1 2; do PPO_MULTISTEP=$v timeout 300 python bench.py --config tiny --steps 50 --warmup 5 > gpurun_out/r2_tiny_ms$v.$i.json 2>&1; done; done
bash tools/scripts/r2_gae_tma2.sh
echo done
