cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/r2_n2_smi.txt
timeout 1200 python -m pytest tests/test_gpu_dp_multi.py tests/test_gpu_dp.py tests/test_gpu_dp_emul.py -q -p no:cacheprovider > gpurun_out/r2_n2_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_n2_tests.txt
for i in 1 2; do
for ov in "" "--no-overlap"; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $ov > gpurun_out/r2_n2_bench$ov.$i.json 2> gpurun_out/r2_n2_bench$ov.$i.err
done; done
echo done
