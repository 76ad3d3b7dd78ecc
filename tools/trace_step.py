"""Phase trace (10 producer exit, 11 MMA-warp exit, 12-15 epilogue warps exit) of the LAST forward step GEMM (EpiLstmFwd, t = T-1) of lstm_bptt_fwd, in an
experiments build with the trace (heads forced onto the single-CTA kernel so they leave the
pair-kernel trace alone):
    PPO_EXPERIMENTS=1 PPO_NVCC_EXTRA=-DPPO_TRACE python paper_1912_06680_b200/build.py
    PPO_VARIANT_HEADS=1cta python tools/trace_step.py --B 32 --H 128 --D 256"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1912_06680_b200 import PPOOptimizer, _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=32)
ap.add_argument("--H", type=int, default=128)
ap.add_argument("--D", type=int, default=256)
ap.add_argument("--mhz", type=float, default=1965.0)
ap.add_argument("--bwd", action="store_true",
                help="trace the last backward step GEMM instead (run with PPO_VARIANT_WGRAD=1cta "
                     "PPO_VARIANT_WGRAD_O=1cta so the weight-gradient GEMMs leave the trace alone)")
a = ap.parse_args()
lib = L._lib
lib.ppo_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
cfg = synth.Config(H=a.H, D=a.D, B=a.B)
opt = PPOOptimizer(a.D, a.H, a.B, 16, cfg.head_sizes, precision="bf16")
p = synth.torch_params(cfg, 0, "cuda")
opt.load_canonical(p["Wx"], p["Wh"], p["b"], p["Wo"], p["bo"])
seq = synth.torch_sequences(cfg, 1, "cuda")
batch = dict(x=seq["x"], h0=seq["h0"], c0=seq["c0"], act=seq["act"], head_on=seq["head_on"],
             avail=seq["avail"])
Lseg = 256 if (a.B * 16) % 256 == 0 else 160
ro = synth.torch_rollouts(a.B * 16 // Lseg, Lseg, 1, "cuda")
batch.update(rew=ro["rew"], val=ro["val"], done=ro["done"])
batch["logp_old"] = opt.current_logp(batch) + seq["logp_noise"]
if a.bwd:
    opt.forward = lambda b: (opt.gae(b), type(opt).forward(opt, b), opt.loss(b), opt.backward())
for _ in range(3):
    opt.forward(batch)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    opt.forward(batch)
e1.record()
torch.cuda.synchronize()
print(f"{'gae+forward+loss+backward' if a.bwd else 'forward (16 step GEMMs + heads)'}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
lib.ppo_trace_clear()
opt.forward(batch)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (512 * 32))()
lib.ppo_trace_read(buf, 512 * 32)
t0s = [buf[32 * b] for b in range(296) if buf[32 * b]]
tmin = min(t0s)
for b in range(12):
    if not buf[32 * b]:
        continue
    ph = [buf[32 * b + i] for i in range(1, 24)]
    print(f"  cta {b:3d} entry +{(buf[32 * b] - tmin) / 1e3:7.2f} us  phases(us @{a.mhz:.0f}): " +
          " ".join(f"{i}:{p / a.mhz:7.2f}" for i, p in zip(range(1, 24), ph) if p))
