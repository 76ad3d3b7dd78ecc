cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > gpurun_out/r2_fine2_build.txt 2>&1 || echo build failed
PPO_MULTISTEP_FINE=1 PPO_MULTISTEP=2 timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_graph.py -x -q -p no:cacheprovider > gpurun_out/r2_fine2_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_fine2_tests.txt
rm -f gpurun_out/r2_fine2_pmb.txt
for r in 1 2; do
for v in "PPO_MULTISTEP_FINE=0" "PPO_MULTISTEP_FINE=1" "PPO_MULTISTEP_FINE=1 PPO_MULTISTEP=2 PPO_MULTISTEP_PERM=0" "PPO_MULTISTEP_FINE=1 PPO_MULTISTEP=2"; do
  echo "== $v" >> gpurun_out/r2_fine2_pmb.txt
  env $v timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print(round(d['value'],1), 'graph', round(d['graph']['ms_per_step'],3), 'eager', round(d['eager']['ms_per_step'],3), 'fwd', round(k['lstm_fwd_step']['us_per_step'],1), 'bwd', round(k['lstm_bwd_step']['us_per_step'],1), d['clocks'])" >> gpurun_out/r2_fine2_pmb.txt 2>&1
done
for v in "PPO_MULTISTEP_FINE=0" "PPO_MULTISTEP_FINE=1"; do
  echo "== tiny $v" >> gpurun_out/r2_fine2_pmb.txt
  env $v timeout 300 python bench.py --config tiny --steps 200 --warmup 20 --no-cpu-baseline 2>/dev/null | tail -1 | grep -o '"value": [0-9.]*' >> gpurun_out/r2_fine2_pmb.txt
done
done
echo done
