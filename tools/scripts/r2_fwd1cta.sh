cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
rm -f gpurun_out/r2_fwd1cta.txt
for r in 1 2; do for B in 600 300; do for v in "PPO_VARIANT_FWD=pair" "PPO_VARIANT_FWD=1cta"; do
  echo "== B=$B $v" >> gpurun_out/r2_fwd1cta.txt
  env $v timeout 300 python bench.py --config paper-mb --small-B $B --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print(round(d['value'],1), 'graph', round(d['graph']['ms_per_step'],3), 'fwd', round(k['lstm_fwd_step']['us_per_step'],1), 'bwd', round(k['lstm_bwd_step']['us_per_step'],1), 'wgrad', round(k['wgrad_xh']['us_per_step'],1), d['roofline']['frac'], d['clocks']['sm_mhz'])" >> gpurun_out/r2_fwd1cta.txt 2>&1
done; done; done
echo done
