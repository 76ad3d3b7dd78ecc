cd $GRAFT_REPO_ROOT
python paper_1912_06680_b200/build.py > /dev/null 2>&1
timeout 2400 bash tools/ab_builds.sh run 3 --steps 10 --warmup 3 > gpurun_out/r2_abb_final3.txt 2>&1
echo done
