cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_graph.py -x -q -p no:cacheprovider > gpurun_out/r2_bsplit_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_bsplit_tests.txt
rm -f gpurun_out/r2_bsplit_pmb.txt
for r in 1 2; do
for v in "PPO_BWD_SPLIT=0" "PPO_BWD_SPLIT=1"; do
  echo "== $v" >> gpurun_out/r2_bsplit_pmb.txt
  env $v timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print(round(d['value'],1), 'graph', round(d['graph']['ms_per_step'],3), 'eager', round(d['eager']['ms_per_step'],3), 'fwd', round(k['lstm_fwd_step']['us_per_step'],1), 'bwd', round(k['lstm_bwd_step']['us_per_step'],1), 'cell', round(k.get('cell_bwd',{}).get('us_per_step',0),1), d['roofline']['frac'], d['clocks'])" >> gpurun_out/r2_bsplit_pmb.txt 2>&1
done
done
for B in 300; do for v in "PPO_BWD_SPLIT=0" "PPO_BWD_SPLIT=1"; do
  echo "== B=$B $v" >> gpurun_out/r2_bsplit_pmb.txt
  env $v timeout 300 python bench.py --config paper-mb --small-B $B --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print(round(d['value'],1), 'graph', round(d['graph']['ms_per_step'],3), 'bwd', round(k['lstm_bwd_step']['us_per_step'],1), 'cell', round(k.get('cell_bwd',{}).get('us_per_step',0),1), d['roofline']['frac'])" >> gpurun_out/r2_bsplit_pmb.txt 2>&1
done; done
echo done
