"""Data-parallel equivalence on real GPUs over NCCL (SURVEY §4b "DP equivalence"): N ranks
each take B/N sequences of one seeded minibatch, the library averages the gradients
(grad_allreduce, ncclAvg) and applies Adam; rank 0 also runs the whole batch alone on its
GPU.  Both gradients and updated parameters must agree (fp32 path: 1e-5 normwise -- the
sum order differs; bf16 path: 2e-2).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        tools/dist_parity.py --precision fp32
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from gpu_util import device_batch, load_params, make_case  # noqa: E402
from paper_1912_06680_b200 import PPOOptimizer  # noqa: E402
from paper_1912_06680_b200 import dist as pdist  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--precision", default="fp32")
ap.add_argument("--dp", default="allreduce", choices=("allreduce", "fused", "fused-push"))
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
rank, world, local = pdist.env()
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
dev = torch.device("cuda", local)
cfg = synth.Config(H=128, D=256, B=64)
case = make_case(cfg, 5, pad_frac=0.2, wo_scale=20.0)   # same seed on every rank
full = device_batch(case, a.precision == "bf16", device=dev)
Bs, Rs = cfg.B // world, case["ro"]["r"].shape[0] // world
sl, rs = slice(rank * Bs, (rank + 1) * Bs), slice(rank * Rs, (rank + 1) * Rs)
shard = {k: (v[:, sl] if k in ("x", "act", "head_on", "avail", "valid", "logp_old")
             else v[sl] if k in ("h0", "c0") else v[rs]).contiguous() for k, v in full.items()}
comm = pdist.make_comm(dev)
opt = PPOOptimizer(cfg.D, cfg.H, Bs, cfg.T, cfg.head_sizes, precision=a.precision, device=dev,
                   comm=comm, n_buckets=4, dp=a.dp)
load_params(opt, case["params"], device=dev)
# each rank's loss uses its local denominator T*Bs (DESIGN Q9), so the average of the N
# gradients is the gradient of the whole batch over T*B
import numpy as np  # noqa: E402

import oracle  # noqa: E402

from gpu_util import HYPER as H  # noqa: E402
orc = {}
for s in range(a.steps):
    th_before = opt.theta.clone() if s == 0 else None
    opt.step(shard)
    if s == 0:
        # after step 1, against the ORACLE on the whole batch (fp64; DESIGN O9/O10): the
        # averaged gradient (allreduce path keeps it), m = (1-b1) clip(g) (every path), and
        # the update where the oracle gradient's sign is resolved by the tolerance
        opt.gather_sharded()
        torch.cuda.synchronize()
        if rank == 0:
            keys = ("Wx", "Wh", "b", "Wo", "bo")
            mo = {k: v.cpu().numpy().astype(np.float64) for k, v in opt.unpack(opt.m).items()}
            new = {k: v.cpu().numpy().astype(np.float64) for k, v in opt.unpack(opt.theta).items()}
            old = {k: v.cpu().numpy().astype(np.float64)
                   for k, v in opt.unpack(th_before).items()}
            gref = case["grads"]
            nwn = lambda x, y: float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300))  # noqa: E731
            cat = lambda d: np.concatenate([np.ravel(d[k]) for k in keys])  # noqa: E731
            m_ref, d_ref, firm = {}, {}, {}
            fp32 = a.precision == "fp32"
            for k in keys:
                z = np.zeros_like(old[k])
                p1, m_ref[k], _ = oracle.adam_clip(old[k], gref[k], z, z, 1, H["lr"], H["beta1"],
                                                   H["beta2"], H["adam_eps"], H["clip_sigma"])
                d_ref[k] = p1 - old[k]
                if fp32:
                    # theta is stored in fp32: ulp(theta) is ~1e-4 of the first update, so the
                    # reference update is the fp32 rounding of old + d_ref (as test_gpu_step)
                    d_ref[k] = (old[k] + d_ref[k]).astype(np.float32).astype(np.float64) - old[k]
                # the first Adam step is ~ -alpha sign(g) times a constant, so compare where
                # the GPU resolves the gradient: m = (1-b1) clip(g) is proportional to the
                # averaged gradient, and its error shows how well each entry is resolved
                # (fp32: to 1e-4 relative, as test_gpu_step; bf16: the sign, 3x)
                firm[k] = np.abs(m_ref[k]) > (1e4 if fp32 else 3.0) * np.abs(mo[k] - m_ref[k]) + \
                    1e-6 * np.abs(m_ref[k]).max()
            orc["oracle_m_err"] = nwn(cat(mo), cat(m_ref))
            dg = cat({k: (new[k] - old[k])[firm[k]] for k in keys})
            dr = cat({k: d_ref[k][firm[k]] for k in keys})
            orc["oracle_update_err"] = nwn(dg, dr)
            orc["oracle_firm_frac"] = float(np.mean(cat(firm)))
            if a.dp == "allreduce":
                go = {k: v.cpu().numpy().astype(np.float64) for k, v in opt.unpack(opt.grad).items()}
                orc["oracle_grad_err"] = nwn(cat(go), cat(gref))
opt.gather_sharded()
torch.cuda.synchronize()
res = {}
if rank == 0:
    ref = PPOOptimizer(cfg.D, cfg.H, cfg.B, cfg.T, cfg.head_sizes, precision=a.precision,
                       device=dev)
    load_params(ref, case["params"], device=dev)
    th0 = ref.theta.clone()
    for _ in range(a.steps):
        ref.step(full)
    torch.cuda.synchronize()
    nw = lambda x, y: float((x - y).norm() / y.norm())  # noqa: E731
    res = {"world": world, "precision": a.precision, "dp": a.dp, "steps": a.steps,
           "theta_err": nw(opt.theta, ref.theta),
           "update_err": nw(opt.theta - th0, ref.theta - th0),
           "m_err": nw(opt.m, ref.m), "v_err": nw(opt.v, ref.v)}
    if a.dp == "allreduce":   # the fused paths leave each rank's own (unaveraged) gradient
        res["grad_err"] = nw(opt.grad, ref.grad)
    tol = 1e-5 if a.precision == "fp32" else 2e-2
    # the oracle bar of north_star: 1e-4 (fp32 path) / 2e-2 (bf16) normwise
    otol = 1e-4 if a.precision == "fp32" else 2e-2
    res.update(orc)
    # the update vs one GPU: differences of fp32 theta values, so one ulp of theta (~1e-4 of
    # the first update) per element whose rounding differs -- the update bar is the oracle's
    res["ok"] = (max(res.get("grad_err", 0.0), res["m_err"], res["v_err"], res["theta_err"]) < tol
                 and res["update_err"] < otol
                 and max(orc["oracle_m_err"], orc["oracle_update_err"],
                         orc.get("oracle_grad_err", 0.0)) < otol
                 and orc["oracle_firm_frac"] > (0.9 if a.precision == "fp32" else 0.8))
    print(json.dumps(res), flush=True)
# every rank holds identical parameters after the averaged update
th = opt.theta.clone()
dist.broadcast(th, 0)
same = bool(torch.equal(th, opt.theta))
if opt.shadow is not None:
    sh = opt.shadow.clone()
    dist.broadcast(sh, 0)
    same = same and bool(torch.equal(sh, opt.shadow))
flag = torch.tensor([1 if same else 0], device=dev)
dist.all_reduce(flag, op=dist.ReduceOp.MIN)
if rank == 0:
    print(json.dumps({"replicas_identical": bool(flag.item())}), flush=True)
from paper_1912_06680_b200 import _lib as L  # noqa: E402
if a.dp == "fused-push" and opt.dp_push:
    # push mode (gradient shards delivered by the backward's epilogues) against pull mode
    # (owners read them after the backward) on a second communicator: the same bits
    comm2 = pdist.make_comm(dev)
    opt2 = PPOOptimizer(cfg.D, cfg.H, Bs, cfg.T, cfg.head_sizes, precision=a.precision,
                        device=dev, comm=comm2, dp="fused")
    load_params(opt2, case["params"], device=dev)
    for _ in range(a.steps):
        opt2.step(shard)
    opt2.gather_sharded()
    torch.cuda.synchronize()
    eq = all(torch.equal(getattr(opt, k), getattr(opt2, k)) for k in ("theta", "m", "v", "grad"))
    if opt.shadow is not None:
        eq = eq and torch.equal(opt.shadow, opt2.shadow)
    flag = torch.tensor([1 if eq else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"push_equals_pull": bool(flag.item())}), flush=True)
    del opt2
    L.comm_destroy(comm2)
L.comm_destroy(comm)
dist.destroy_process_group()
