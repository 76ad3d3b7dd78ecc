cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/r2_tiny_launches.csv python tools/profile_step.py --B 32 --H 128 --D 256 --steps 1 --warmup 1 > gpurun_out/r2_tiny_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --kernel-name regex:EpiLstmFwd --launch-skip 20 --launch-count 1 -o gpurun_out/r2_tiny_fwd python tools/profile_step.py --B 32 --H 128 --D 256 --steps 1 --warmup 1 >> gpurun_out/r2_tiny_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_pmb_launches.csv python tools/profile_step.py --B 600 --steps 1 --warmup 1 > gpurun_out/r2_pmb_ncu.log 2>&1
echo done
