# usage: bash tools/scripts/dp_ab3.sh N ROUNDS -- interleaved bench A/B: fused (pull), fused-push, nccl
N=${1:-2}; R=${2:-2}
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for r in $(seq 1 $R); do
  for dp in fused fused-push nccl; do
    timeout 900 $TR --master-port 2957$N bench.py --gpus $N --steps 8 --warmup 3 --no-e2e --dp $dp > gpurun_out/ab3_${dp}_n${N}_$r.json 2> gpurun_out/ab3_${dp}_n${N}_$r.err
    echo -n "$dp r$r rc=$? "
    python tools/scripts/bench_brief.py gpurun_out/ab3_${dp}_n${N}_$r.json
  done
done
