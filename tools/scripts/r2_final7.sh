cd $GRAFT_REPO_ROOT
python paper_1912_06680_b200/build.py > gpurun_out/r2_final7_build.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2_final7_smi.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_final7_gpu_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_final7_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_final7_smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/r2_final7_smoke.txt
timeout 900 python bench.py > gpurun_out/r2_final7_bench.json 2> gpurun_out/r2_final7_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2_final7_ref.json 2> gpurun_out/r2_final7_ref.err
timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 > gpurun_out/r2_final7_pmb.json 2> gpurun_out/r2_final7_pmb.err
timeout 300 python bench.py --config tiny --steps 50 --warmup 5 > gpurun_out/r2_final7_tiny.json 2> gpurun_out/r2_final7_tiny.err
timeout 600 python bench.py --config gae > gpurun_out/r2_final7_gae.json 2> gpurun_out/r2_final7_gae.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_final7_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2_final7_launches_ncu.log 2>&1
echo done
