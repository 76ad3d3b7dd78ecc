cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py -q -p no:cacheprovider -k "tc_gemm or step or fullsize" > gpurun_out/r2_t3_tests.txt 2>&1
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 900 python tools/ab_variants.py --B 38400 --var PPO_DIE_SCHED --vals 0,1 --rounds 3 --steps 3 > gpurun_out/r2_ab_die.txt 2>&1
for v in 0 1; do
PPO_DIE_SCHED=$v timeout 600 ncu --set full --clock-control none --kernel-name regex:"EpiLstmFwd|EpiLstmBwd|tc_gemm2_kernel<1, 1, 4, 2" --launch-skip 40 --launch-count 6 -o gpurun_out/r2_die$v python tools/profile_step.py --B 38400 --steps 1 --warmup 1 > gpurun_out/r2_die_ncu$v.log 2>&1
done
echo done
