cd $GRAFT_REPO_ROOT
bash tools/ab_builds.sh run 3 --steps 4 --warmup 2 > gpurun_out/r2_bisect.txt 2>&1
echo done
