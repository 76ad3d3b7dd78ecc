cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 1200 python tools/ab_variants.py --B 38400 --var PPO_GRID_ALL_TILES_wgrad_xh --vals 0,1 --rounds 3 --steps 3 > gpurun_out/r2_ab_wgrad_alltiles.txt 2>&1
for v in 0 1; do
PPO_GRID_ALL_TILES_wgrad_xh=$v timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_ltcfabric.sum --clock-control none --kernel-name-base demangled --kernel-name regex:"tc_gemm2_kernel<1, 1, 4, 2" --launch-skip 4 --launch-count 2 --csv python tools/profile_step.py --B 38400 --steps 1 --warmup 1 > gpurun_out/r2_wgrad_alltiles_ncu$v.csv 2>&1
done
echo done
