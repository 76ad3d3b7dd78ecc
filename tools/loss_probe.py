"""Time ppo_loss_grad alone at the bench shape (T=16, B=38400, the paper's 7 heads + value),
device-generated inputs, CUDA events over --reps back-to-back launches.
    python tools/loss_probe.py [--lib-root DIR] [--B 38400] [--fp32]"""
import argparse
import os
import sys

ap = argparse.ArgumentParser()
ap.add_argument("--lib-root", default=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap.add_argument("--B", type=int, default=38400)
ap.add_argument("--T", type=int, default=16)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--fp32", action="store_true")
a = ap.parse_args()
sys.path.insert(0, a.lib_root)
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1912_06680_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda")
cfg = synth.Config(H=128, D=128, B=a.B, T=a.T)
s = synth.torch_sequences(cfg, 3, dev)
N = a.T * a.B
A = sum(cfg.head_sizes) + 1
out = torch.randn((N, A), device=dev) * 2.0
prec = L.PPO_PREC_FP32 if a.fp32 else L.PPO_PREC_BF16
dims = L.make_dims(cfg.D, cfg.H, cfg.T, cfg.head_sizes, prec)
lc = L.ppo_loss_cfg(0.2, 0.5, 0.01, float(N), 0.0, 0.0, 0.0)
dout = torch.empty((N, A), device=dev, dtype=torch.float32 if a.fp32 else torch.bfloat16)
logp = torch.empty(N, device=dev)
stats = torch.zeros(L.PPO_STATS_BUF, device=dev)
lo = torch.randn(N, device=dev) - 8.0
adv, ret = torch.randn(N, device=dev), torch.randn(N, device=dev)
valid = (torch.rand(N, device=dev) < 0.95).to(torch.uint8)
f = lambda: L.ppo_loss_grad(dims, out, s["act"], s["head_on"], s["avail"], lo, adv, ret, valid,
                            a.B, lc, dout, logp, stats)
for _ in range(3):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
nb = N * (A * (4 + dout.element_size()) + 7 * 4 + 7 + 30 + 1 + 4 * 4)
print(f"{L.LIB_PATH}: loss ms={ms:.4f} GB/s(alg)={nb / ms / 1e6:.0f} "
      f"dsum={dout.float().abs().sum().item():.6e} stats={[round(v, 6) for v in stats[:8].tolist()]}",
      flush=True)
