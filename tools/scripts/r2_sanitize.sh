cd $GRAFT_REPO_ROOT
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_tiny.py > gpurun_out/r2_sanitize_memcheck.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_sanitize_memcheck.txt
echo done
