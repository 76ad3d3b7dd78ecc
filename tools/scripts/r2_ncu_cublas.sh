# ncu --set full of cuBLAS vs the tcgen05 kernels on the step's GEMM shapes (GEMM launches only)
cd $GRAFT_REPO_ROOT
for s in fwd bwd wgrad; do
  timeout 600 ncu --set full --clock-control none --kernel-name regex:"nvjet|gemm|cutlass|sm100|xmma|Kernel" -c 4 -o gpurun_out/r2_cmp_$s python tools/gemm_one.py $s > gpurun_out/r2_cmp_$s.log 2>&1
done
echo done
