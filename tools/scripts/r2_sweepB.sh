cd $GRAFT_REPO_ROOT
python paper_1912_06680_b200/build.py > /dev/null 2>&1
rm -f gpurun_out/r2_sweepB.jsonl
for B in 2400 9600 19200 38400 76800 123648; do
  st=5; [ $B -ge 76800 ] && st=3
  timeout 900 python bench.py --B $B --steps $st --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print(json.dumps({'B': $B, 'samples_per_s': d['value'], 'ms_per_step': d['ms_per_step'], 'sm_mhz': d['clocks']['sm_mhz'], 'step_frac': d['roofline']['step']['frac'], 'dominant': d['roofline']['kernel'], 'dominant_frac': d['roofline']['frac'], 'bwd_frac': k['lstm_bwd_step']['frac'], 'fwd_frac': k['lstm_fwd_step']['frac']}))" >> gpurun_out/r2_sweepB.jsonl
done
timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(json.dumps({'B': 600, 'samples_per_s': d['value'], 'ms_per_step': d['ms_per_step'], 'sm_mhz': d['clocks']['sm_mhz'], 'gemm_frac': d['roofline']['frac'], 'graph': True}))" >> gpurun_out/r2_sweepB.jsonl
echo done
