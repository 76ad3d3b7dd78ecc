"""Time ppo_gae for a list of rollout lengths at ~N total timesteps (HBM GB/s, 17 B/step).
    python tools/gae_probe.py --L 1280,1344,1350 --steps 1000000000"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1912_06680_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--L", default="256,1280,1344,1350,1536,6300,20000,1000000")
ap.add_argument("--steps", type=int, default=10 ** 9)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--seq-T", type=int, default=0)
a = ap.parse_args()
dev = torch.device("cuda")
gamma = 1.0 - (4.0 / 30.0) / 180.0
for Lr in (int(x) for x in a.L.split(",")):
    R = max(1, a.steps // Lr)
    n = R * Lr
    ro = synth.torch_rollouts(R, Lr, 1, dev)
    adv = torch.empty((R, Lr), device=dev)
    ret = torch.empty((R, Lr), device=dev)
    nb = L.gae_scratch_bytes(R, Lr)
    scratch = torch.empty(nb, dtype=torch.uint8, device=dev) if nb else None
    f = lambda: L.ppo_gae(ro["rew"], ro["val"], ro["done"], gamma, 0.95, adv, ret,
                          seq_T=a.seq_T, scratch=scratch)
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    print(f"L={Lr:8d} R={R:9d} ms={ms:8.3f} GB/s={17.0 * n / ms / 1e6:8.1f}", flush=True)
    del ro, adv, ret, scratch
    torch.cuda.empty_cache()
