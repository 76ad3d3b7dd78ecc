"""Run a few PPO steps at a chosen minibatch size (for ncu captures and quick timing).

    python tools/profile_step.py --B 9600 --steps 2
Prints the per-kernel device time from the library's tracing hooks."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1912_06680_b200 import PPOOptimizer, _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=9600)
ap.add_argument("--H", type=int, default=4096)
ap.add_argument("--D", type=int, default=4032)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--warmup", type=int, default=1)
a = ap.parse_args()
cfg = synth.Config(H=a.H, D=a.D, B=a.B)
opt = PPOOptimizer(a.D, a.H, a.B, 16, cfg.head_sizes, precision="bf16")
p = synth.torch_params(cfg, 0, "cuda")
opt.load_canonical(p["Wx"], p["Wh"], p["b"], p["Wo"], p["bo"])
seq = synth.torch_sequences(cfg, 1, "cuda")
Lseg = 256 if (a.B * 16) % 256 == 0 else 160   # B = 600: 60 segments of 160 steps
ro = synth.torch_rollouts(a.B * 16 // Lseg, Lseg, 1, "cuda")
batch = dict(x=seq["x"], h0=seq["h0"], c0=seq["c0"], act=seq["act"], head_on=seq["head_on"],
             avail=seq["avail"], rew=ro["rew"], val=ro["val"], done=ro["done"])
batch["logp_old"] = opt.current_logp(batch) + seq["logp_noise"]
for _ in range(a.warmup):
    opt.step(batch)
torch.cuda.synchronize()
L.prof_start()
for _ in range(a.steps):
    opt.step(batch)
torch.cuda.synchronize()
prof = L.prof_stop()
tot = sum(ms for _, ms in prof.values())
for k, (n, ms) in prof.items():
    print(f"{k:16s} launches {n:5d}  ms/step {ms / a.steps:9.3f}  share {ms / tot:6.3f}")
print("stats", dict(zip(L.STAT_NAMES, opt.stats[:8].tolist())))
