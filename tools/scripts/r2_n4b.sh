cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/r2_n4b_smi.txt
timeout 1200 python -m pytest tests/test_gpu_dp_multi.py -q -p no:cacheprovider > gpurun_out/r2_n4b_dp_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_n4b_dp_tests.txt
for dp in allreduce fused; do for prec in fp32 bf16; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741 tools/dist_parity.py --precision $prec --dp $dp --steps 2 >> gpurun_out/r2_n4b_parity.txt 2>&1
done; done
for rep in 1 2; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_n4b_bench_n1.$rep.json 2> /dev/null
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29742 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_n4b_bench_n2.$rep.json 2> /dev/null
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29743 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_n4b_bench_n4.$rep.json 2> /dev/null
done
echo done
