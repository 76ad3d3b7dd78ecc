"""BASELINE configs[1]/[4]: PPO step throughput vs per-GPU minibatch B (sequences), up to the
largest B whose workspace fits in HBM.

    python tools/sweep_B.py [--Bs 600,2400,9600,38400,76800] [--max]
Prints one JSON line per B (device-timed, CUDA events, inputs resident)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1912_06680_b200 import PPOOptimizer, _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--Bs", default="640,2560,9600,38400,76800")
ap.add_argument("--max", action="store_true", help="also the largest B that fits")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=2)
a = ap.parse_args()
H, D, T = 4096, 4032, 16
heads = synth.HEAD_SIZES


def bytes_per_seq():
    dims = L.make_dims(D, H, T, heads)
    ws = L.ws_bytes(dims, 1024) / 1024
    inputs = T * D * 2 + 2 * H * 4 + T * (7 * 4 + 7 + 30 + 4) + 256 / T * 9
    outs = T * synth.A_OUT * (4 + 2) + T * 4 * 3
    return ws + inputs + outs


def run(B):
    cfg = synth.Config(H=H, D=D, B=B)
    opt = PPOOptimizer(D, H, B, T, heads, precision="bf16")
    p = synth.torch_params(cfg, 0, "cuda")
    opt.load_canonical(p["Wx"], p["Wh"], p["b"], p["Wo"], p["bo"])
    del p
    seq = synth.torch_sequences(cfg, 1, "cuda")
    ro = synth.torch_rollouts(B * T // 256, 256, 1, "cuda")
    batch = dict(x=seq["x"], h0=seq["h0"], c0=seq["c0"], act=seq["act"], head_on=seq["head_on"],
                 avail=seq["avail"], rew=ro["rew"], val=ro["val"], done=ro["done"])
    batch["logp_old"] = opt.current_logp(batch) + seq["logp_noise"]
    for _ in range(a.warmup):
        opt.step(batch)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        opt.step(batch)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    flop = B * 2.0 * T * 4 * H * (2 * D + 3 * H) + B * 6.0 * T * H * synth.A_OUT
    out = dict(B=B, paper_samples=B // 5, ms_per_step=ms, samples_per_s=B / 5 / (ms / 1e3),
               sequences_per_s=B / (ms / 1e3), tflops=flop / (ms / 1e3) / 1e12,
               mem_gb=torch.cuda.max_memory_allocated() / 1e9)
    print(json.dumps(out), flush=True)
    del opt, batch, seq, ro
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()


Bs = [int(x) for x in a.Bs.split(",") if x]
if a.max:
    free, total = torch.cuda.mem_get_info()
    bmax = int((free - 6e9) / bytes_per_seq()) // 256 * 256
    Bs.append(bmax)
for B in Bs:
    run(B)
