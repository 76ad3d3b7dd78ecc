cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 1500 python tools/ab_variants.py --B 38400 --steps 3 --rounds 3 --var PPO_WGRAD_CHUNK --vals 153600,307200,614400 > gpurun_out/r2_chunk_ab.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_chunk_ab.txt
echo done
