cd $GRAFT_REPO_ROOT
for Lr in 1350 1000000; do
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled --kernel-name regex:gae --launch-skip 1 --launch-count 1 -o gpurun_out/r2_gae_$Lr python tools/gae_probe.py --L $Lr --reps 1 > gpurun_out/r2_gae_ncu_$Lr.log 2>&1
done
echo done
