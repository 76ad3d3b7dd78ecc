cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_graph.py tests/test_gpu_aux.py tests/test_gpu_trainer.py -q -p no:cacheprovider -x > gpurun_out/r2_t6_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_t6_tests.txt
timeout 300 python bench.py --config tiny --steps 50 --warmup 5 > gpurun_out/r2_tiny.json 2> gpurun_out/r2_tiny.err
timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 > gpurun_out/r2_pmb.json 2> gpurun_out/r2_pmb.err
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
for v in 0 1; do PPO_MULTISTEP=$v timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 > gpurun_out/r2_pmb_ms$v.json 2>&1; done
timeout 900 python tools/ab_variants.py --B 38400 --var PPO_DIE_SCHED --vals 0,1 --rounds 3 --steps 3 > gpurun_out/r2_ab_die2.txt 2>&1
for v in 0 1; do
PPO_DIE_SCHED=$v timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_ltcfabric.sum --clock-control none --kernel-name-base demangled --kernel-name regex:"EpiLstmFwd|EpiLstmBwd|tc_gemm2_kernel<1, 1, 4, 2" --launch-skip 40 --launch-count 6 --csv python tools/profile_step.py --B 38400 --steps 1 --warmup 1 > gpurun_out/r2_die_ncu$v.csv 2>&1
done
echo done
