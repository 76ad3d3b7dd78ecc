"""A/B the GEMM kernel variants in one process on one GPU (alternating rounds), with the
library's per-kernel event timing and nvidia-smi clocks/power per round.

    python tools/ab_variants.py --B 38400 --var PPO_TC_PAIR --vals 1,0
"""
import argparse
import os
import subprocess
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1912_06680_b200 import PPOOptimizer, _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=38400)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("--var", default="PPO_TC_PAIR")
ap.add_argument("--vals", default="1,0")
a = ap.parse_args()
cfg = synth.Config(H=4096, D=4032, B=a.B)
opt = PPOOptimizer(4032, 4096, a.B, 16, cfg.head_sizes, precision="bf16")
p = synth.torch_params(cfg, 0, "cuda")
opt.load_canonical(p["Wx"], p["Wh"], p["b"], p["Wo"], p["bo"])
del p
seq = synth.torch_sequences(cfg, 1, "cuda")
ro = synth.torch_rollouts(a.B * 16 // 256, 256, 1, "cuda")
batch = dict(x=seq["x"], h0=seq["h0"], c0=seq["c0"], act=seq["act"], head_on=seq["head_on"],
             avail=seq["avail"], rew=ro["rew"], val=ro["val"], done=ro["done"])
batch["logp_old"] = opt.current_logp(batch) + seq["logp_noise"]
opt.step(batch)
torch.cuda.synchronize()


pynvml.nvmlInit()
_nv = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())


def smi():
    q = "clocks.sm,power.draw"
    proc = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={q}",
                             "--format=csv,noheader,nounits", "-lms", "100"],
                            stdout=subprocess.PIPE, text=True)
    lines = []
    t = threading.Thread(target=lambda: lines.extend(l.strip() for l in proc.stdout), daemon=True)
    t.start()
    return proc, lines


def med(z):
    return z[len(z) // 2] if z else float("nan")


for r in range(a.rounds):
    for v in a.vals.split(","):
        os.environ[a.var] = v
        opt.step(batch)
        torch.cuda.synchronize()
        proc, lines = smi()
        L.prof_start()
        j0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(_nv)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            opt.step(batch)
        e1.record()
        torch.cuda.synchronize()
        j1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(_nv)
        prof = L.prof_stop()
        proc.terminate()
        vals = []
        for ln in lines:
            try:
                vals.append(tuple(float(x) for x in ln.split(",")))
            except ValueError:
                pass
        clk = sorted(x[0] for x in vals)
        pw = sorted(x[1] for x in vals)
        ms = e0.elapsed_time(e1) / a.steps
        ks = " ".join(f"{k}={prof[k][1] / a.steps:.1f}"
                      for k in ("lstm_fwd_step", "lstm_bwd_step", "wgrad_xh") if k in prof)
        print(f"round {r} {a.var}={v}: step {ms:.1f} ms  {(j1 - j0) / 1e3 / a.steps:.1f} J/step  "
              f"sm_mhz~{med(clk):.0f} power~{med(pw):.0f}W  {ks}", flush=True)
