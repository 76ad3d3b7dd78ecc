"""Time adam_step alone on the full parameter vector (135.9 M fp32 + bf16 shadow), CUDA
events over --reps launches; algorithmic 30 B/param.
    python tools/adam_probe.py [--lib-root DIR] [--n N]"""
import argparse
import os
import sys

ap = argparse.ArgumentParser()
ap.add_argument("--lib-root", default=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap.add_argument("--n", type=int, default=135_917_728)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
sys.path.insert(0, a.lib_root)
import torch  # noqa: E402

from paper_1912_06680_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda")
p = torch.randn(a.n, device=dev)
g = torch.randn(a.n, device=dev) * 1e-3
m = torch.zeros(a.n, device=dev)
v = torch.zeros(a.n, device=dev)
sh = torch.empty(a.n, dtype=torch.bfloat16, device=dev)
f = lambda t: L.adam_step(p, sh, g, m, v, t, 5e-5, 0.9, 0.999, 1e-8, 5.0)  # noqa: E731
for t in range(1, 4):
    f(t)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for t in range(4, 4 + a.reps):
    f(t)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
print(f"{L.LIB_PATH}: adam ms={ms:.4f} GB/s(alg)={30.0 * a.n / ms / 1e6:.0f} "
      f"psum={p.double().sum().item():.6e}", flush=True)
