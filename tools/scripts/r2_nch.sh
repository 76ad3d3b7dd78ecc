cd $GRAFT_REPO_ROOT
PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_graph.py tests/test_gpu_aux.py tests/test_gpu_dp.py -q -x -p no:cacheprovider > gpurun_out/r2_nch_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_nch_tests.txt
rm -f gpurun_out/r2_nch_tiny.txt
for r in 1 2; do for b in 1 2; do
  echo "== build $b ($(cat .ab/$b/REV))" >> gpurun_out/r2_nch_tiny.txt
  (cd .ab/$b && [ -f paper_1912_06680_b200/libppo5.so ] || python paper_1912_06680_b200/build.py > /dev/null 2>&1)
  PPO_LIB_PATH=$PWD/.ab/$b/paper_1912_06680_b200/libppo5.so timeout 300 python bench.py --config tiny --steps 200 --warmup 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print(round(d['value'],1), 'us/step graph; fwd', round(k['lstm_fwd_step']['us_per_step'],1), 'bwd', round(k['lstm_bwd_step']['us_per_step'],1))" >> gpurun_out/r2_nch_tiny.txt 2>&1
done; done
python paper_1912_06680_b200/build.py > /dev/null 2>&1
timeout 2400 bash tools/ab_builds.sh run 3 --steps 10 --warmup 3 > gpurun_out/r2_nch_ab.txt 2>&1
echo done
