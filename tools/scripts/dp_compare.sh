# usage: bash tools/scripts/dp_compare.sh N  -- DP parity (fused and allreduce exchange) and
# bench lines for both at N GPUs; outputs under gpurun_out/
N=${1:-2}
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for prec in fp32 bf16; do
  for dp in fused fused-push allreduce; do
    timeout 300 $TR --master-port 2951$N tools/dist_parity.py --precision $prec --dp $dp --steps 2 2>&1 | grep '^{'
  done
done
for dp in fused fused-push nccl; do
  timeout 900 $TR --master-port 2952$N bench.py --gpus $N --steps 6 --warmup 3 --no-e2e --dp $dp > gpurun_out/bench_dp_${dp}_n$N.json 2> gpurun_out/bench_dp_${dp}_n$N.err
  echo "$dp rc=$?"
  python tools/scripts/bench_brief.py gpurun_out/bench_dp_${dp}_n$N.json
done
