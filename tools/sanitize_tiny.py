"""The tiny configs of every ABI call in one process, for compute-sanitizer
(memcheck / racecheck / synccheck), SURVEY §4b:

    compute-sanitizer --tool memcheck python tools/sanitize_tiny.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from gpu_util import AUX_HYPER, dev, device_batch, load_params, make_case  # noqa: E402
from paper_1912_06680_b200 import PPOOptimizer, _lib as L  # noqa: E402
from paper_1912_06680_b200.infer import PolicyServer  # noqa: E402

# the step, both precisions, ragged B, with aux heads and dL/dx
for precision in ("bf16", "fp32"):
    cfg = synth.Config(H=128, D=192, B=48, aux=synth.AUX_SIZES)
    case = make_case(cfg, 1, pad_frac=0.2, wo_scale=10.0, aux_hyper=AUX_HYPER)
    opt = PPOOptimizer(cfg.D, cfg.H, cfg.B, cfg.T, cfg.head_sizes, precision=precision,
                       aux=cfg.aux, hyper=AUX_HYPER)
    load_params(opt, case["params"])
    dx = torch.empty(cfg.T, cfg.B, cfg.D, device="cuda")
    opt.step(device_batch(case, precision == "bf16"), dx=dx)
    torch.cuda.synchronize()
    print(precision, "step ok", opt.stats[:L.PPO_STATS].cpu().numpy())
# GAE: warp kernel (both chunk sizes) and the look-back kernel
for R, Lr in ((3, 300), (700, 300), (2, 20000)):
    ro = synth.torch_rollouts(R, Lr, 1, "cuda")
    adv = torch.empty(R, Lr, device="cuda")
    ret = torch.empty(R, Lr, device="cuda")
    nb = L.gae_scratch_bytes(R, Lr)
    scratch = torch.empty(nb, dtype=torch.uint8, device="cuda") if nb else None
    L.ppo_gae(ro["rew"], ro["val"], ro["done"], 0.999, 0.95, adv, ret, scratch=scratch)
torch.cuda.synchronize()
print("gae ok")
# the inference step
cfg = synth.Config(H=128, D=128, B=40, T=1)
srv = PolicyServer(cfg.D, cfg.H, cfg.B, cfg.head_sizes)
opt = PPOOptimizer(cfg.D, cfg.H, cfg.B, 1, cfg.head_sizes, precision="bf16")
p = synth.make_params(cfg, 2, bo_scale=0.1)
load_params(opt, p)
srv.load(opt.shadow)
s = synth.make_sequences(cfg, 3)
srv.reset(dev(s["h0"]), dev(s["c0"]))
for t in range(2):
    srv.step(dev(s["x"][0]).bfloat16(), dev(s["avail"][0]))
torch.cuda.synchronize()
print("infer ok", srv.act[0].cpu().numpy())
