cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
rm -f gpurun_out/r2_gae_wpb.txt
for r in 1 2; do for v in 4 2 1; do echo "wpb $v" >> gpurun_out/r2_gae_wpb.txt; PPO_GAE_WPB=$v timeout 300 python tools/gae_probe.py --L 100000,1000000 --steps 1000000000 >> gpurun_out/r2_gae_wpb.txt 2>&1; done; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gae_tma --launch-skip 1 --launch-count 1 -o gpurun_out/r2_gae_l1e6 -f python tools/gae_probe.py --L 1000000 --steps 1000000000 --reps 1 > gpurun_out/r2_gae_ncu.log 2>&1
echo done
