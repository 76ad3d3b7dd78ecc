cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/die_probe tools/cuda/die_probe.cu && /tmp/die_probe > gpurun_out/r2_die_probe.txt 2>&1
/tmp/die_probe >> gpurun_out/r2_die_probe.txt 2>&1
timeout 300 python bench.py --config tiny --steps 50 --warmup 5 > gpurun_out/r2_tiny.json 2> gpurun_out/r2_tiny.err
timeout 300 python bench.py --config paper-mb --steps 30 --warmup 5 > gpurun_out/r2_pmb.json 2> gpurun_out/r2_pmb.err
echo done
