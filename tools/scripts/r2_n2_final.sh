cd $GRAFT_REPO_ROOT
python paper_1912_06680_b200/build.py > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_dp_multi.py tests/test_gpu_dp.py tests/test_gpu_dp_emul.py -q -p no:cacheprovider > gpurun_out/r2_n2_final_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/r2_n2_final_tests.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29751 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2_n2_final_bench.json 2> gpurun_out/r2_n2_final_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29752 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/r2_n2_final_ref.json 2> gpurun_out/r2_n2_final_ref.err
echo done
