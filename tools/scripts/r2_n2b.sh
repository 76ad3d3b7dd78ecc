cd $GRAFT_REPO_ROOT
for dp in allreduce fused; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29721 tools/dist_parity.py --precision fp32 --dp $dp --steps 2 >> gpurun_out/r2_n2_parity.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29722 tools/dist_parity.py --precision bf16 --dp $dp --steps 2 >> gpurun_out/r2_n2_parity.txt 2>&1
done
echo done
