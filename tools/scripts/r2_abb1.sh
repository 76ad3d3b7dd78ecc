cd $GRAFT_REPO_ROOT
bash tools/ab_builds.sh run 3 --steps 5 --warmup 3 > gpurun_out/r2_abb_r1_vs_head.txt 2>&1
echo done
