cd $GRAFT_REPO_ROOT
python paper_1912_06680_b200/build.py > /dev/null 2>&1
for b in 1 2 3; do (cd .ab/$b && PPO_NVCC_EXTRA="$(cat FLAGS)" python paper_1912_06680_b200/build.py > build.log 2>&1) || echo "build $b failed"; done
rm -f gpurun_out/r2_signal.txt
for r in 1 2 3; do for b in 1 2 3; do
  echo "== build $b ($(cat .ab/$b/FLAGS)) round $r" >> gpurun_out/r2_signal.txt
  PPO_LIB_PATH=$PWD/.ab/$b/paper_1912_06680_b200/libppo5.so timeout 300 python bench.py --config tiny --steps 200 --warmup 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('tiny', round(d['value'],1), 'us; fwd', round(k['lstm_fwd_step']['us_per_step'],1), 'bwd', round(k['lstm_bwd_step']['us_per_step'],1))" >> gpurun_out/r2_signal.txt 2>&1
  PPO_LIB_PATH=$PWD/.ab/$b/paper_1912_06680_b200/libppo5.so timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('pmb', round(d['value'],1), 'graph ms', round(d['graph']['ms_per_step'],3), 'fwd', round(k['lstm_fwd_step']['us_per_step'],1), 'bwd', round(k['lstm_bwd_step']['us_per_step'],1))" >> gpurun_out/r2_signal.txt 2>&1
done; done
echo done
