cd $GRAFT_REPO_ROOT
PPO_NVCC_EXTRA="-DPPO_TRACE" python paper_1912_06680_b200/build.py > /dev/null 2>&1 || echo build failed
timeout 300 python tools/trace_gemm.py > gpurun_out/r2_trace.txt 2>&1
python paper_1912_06680_b200/build.py > /dev/null 2>&1
timeout 300 python tools/gae_probe.py --L 256,1350,6300,20000,1000000 --steps 1000000000 > gpurun_out/r2_gae.txt 2>&1
echo done
