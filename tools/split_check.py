"""Diagnostic: the bf16 step on a small-minibatch case with the split-K backward (default) and
the fused-epilogue backward (PPO_BWD_SPLIT=0, experiment builds), against the oracle:
normwise gradient error and the share of entries whose sign is resolved, per tensor.
    PPO_EXPERIMENTS=1 python paper_1912_06680_b200/build.py
    python tools/split_check.py [--H 2048 --D 512 --B 288 --seed 9 --wo 8]"""
import argparse
import os
import subprocess
import sys

here = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(here))
sys.path.insert(0, os.path.join(os.path.dirname(here), "tests"))

ap = argparse.ArgumentParser()
ap.add_argument("--H", type=int, default=2048)
ap.add_argument("--D", type=int, default=512)
ap.add_argument("--B", type=int, default=288)
ap.add_argument("--seed", type=int, default=9)
ap.add_argument("--wo", type=float, default=8.0)
ap.add_argument("--child", action="store_true")
a = ap.parse_args()

if not a.child:
    for v in ("1", "0"):
        env = dict(os.environ, PPO_BWD_SPLIT=v)
        print(f"== PPO_BWD_SPLIT={v}", flush=True)
        subprocess.run([sys.executable, __file__, "--child", "--H", str(a.H), "--D", str(a.D),
                        "--B", str(a.B), "--seed", str(a.seed), "--wo", str(a.wo)], env=env)
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from gpu_util import device_batch, load_params, make_case, normwise  # noqa: E402
from paper_1912_06680_b200 import PPOOptimizer  # noqa: E402

cfg = synth.Config(H=a.H, D=a.D, B=a.B)
case = make_case(cfg, a.seed, pad_frac=0.1, wo_scale=a.wo)
opt = PPOOptimizer(cfg.D, cfg.H, cfg.B, cfg.T, cfg.head_sizes, precision="bf16")
load_params(opt, case["params"])
opt.step(device_batch(case, True))
torch.cuda.synchronize()
g = {k: v.cpu().numpy() for k, v in opt.unpack(opt.grad).items()}
for k in ("Wx", "Wh", "b", "Wo", "bo"):
    ref = case["grads"][k]
    err = np.abs(g[k] - ref)
    firm = np.abs(ref) > 3 * err + 1e-6
    print(f"  {k}: normwise {normwise(g[k], ref):.3e}  sign-resolved {firm.mean():.4f}", flush=True)
