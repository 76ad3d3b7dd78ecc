cd $GRAFT_REPO_ROOT
python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 600 python bench.py --config infer > gpurun_out/r2_sec_infer.json 2> gpurun_out/r2_sec_infer.err
timeout 900 python bench.py --config iteration > gpurun_out/r2_sec_iteration.json 2> gpurun_out/r2_sec_iteration.err
timeout 900 python bench.py --aux --dx --no-cpu-baseline > gpurun_out/r2_sec_auxdx.json 2> gpurun_out/r2_sec_auxdx.err
timeout 900 python bench.py --H 2048 --no-cpu-baseline > gpurun_out/r2_sec_h2048.json 2> gpurun_out/r2_sec_h2048.err
timeout 600 python bench.py --B 123648 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_sec_bmax.json 2> gpurun_out/r2_sec_bmax.err
echo done
