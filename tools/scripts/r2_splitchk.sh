cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 900 python tools/split_check.py > gpurun_out/r2_splitchk.txt 2>&1
timeout 900 python tools/split_check.py --H 4096 --D 4032 --B 48 --seed 7 --wo 5 >> gpurun_out/r2_splitchk.txt 2>&1
echo done
