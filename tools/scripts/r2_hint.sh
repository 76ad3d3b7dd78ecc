cd $GRAFT_REPO_ROOT
for h in 1000000 20000 2000 0; do
  PPO_NVCC_EXTRA="-DPPO_SUSPEND_HINT_NS=$h" python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
  echo "hint $h" >> gpurun_out/r2_hint.txt
  timeout 300 python bench.py --config tiny --steps 30 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('tiny', d['value'], d['eager'], {k: round(v['us_per_step'],1) for k,v in d['kernels'].items()})" >> gpurun_out/r2_hint.txt
  timeout 300 python bench.py --config paper-mb --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pmb', d['value'], d['graph'], d['clocks'], {k: round(v['us_per_step'],1) for k,v in d['kernels'].items()})" >> gpurun_out/r2_hint.txt
done
echo done
python paper_1912_06680_b200/build.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled --kernel-name regex:EpiLstmFwd --launch-skip 20 --launch-count 1 -o gpurun_out/r2_tiny_fwd python tools/profile_step.py --B 32 --H 128 --D 256 --steps 1 --warmup 1 > gpurun_out/r2_tiny_ncu2.log 2>&1
echo done2
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
for v in 0 1; do
PPO_DIE_SCHED=$v timeout 600 ncu --set full --clock-control none --kernel-name-base demangled --kernel-name regex:"EpiLstmFwd|EpiLstmBwd|tc_gemm2_kernel<1, 1, 4, 2" --launch-skip 40 --launch-count 6 -o gpurun_out/r2_die$v python tools/profile_step.py --B 38400 --steps 1 --warmup 1 > gpurun_out/r2_die_ncu$v.log 2>&1
done
echo done3
