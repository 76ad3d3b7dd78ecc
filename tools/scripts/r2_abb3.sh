cd $GRAFT_REPO_ROOT
bash tools/ab_builds.sh run 4 --steps 4 --warmup 2 > gpurun_out/r2_abb3.txt 2>&1
echo done
