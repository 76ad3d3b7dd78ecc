# ncu --set full of one launch of every kernel class of the step at B = 38,400 (final round-2 tree)
cd $GRAFT_REPO_ROOT
run() {  # tag regex skip
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    --kernel-name regex:"$2" --launch-skip $3 --launch-count 1 -o gpurun_out/r2f_tr_$1 \
    python tools/profile_step.py --B 38400 --steps 1 --warmup 1 > gpurun_out/r2f_tr_$1.log 2>&1
}
run lstm_fwd_step "EpiLstmFwd" 20
run heads_fwd "\(int\)224" 1
run lstm_bwd_step "EpiLstmBwd" 20
run wgrad_xh "\(int\)4, \(int\)2" 5
run wgrad_o "\(bool\)1, \(bool\)1, \(int\)6" 1
run loss "loss_fast" 1
run adam "adam_kernel" 1
run gae "gae_kernel" 1
run pack_state "pack_state" 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2f_launches_ncu.log 2>&1
echo done
