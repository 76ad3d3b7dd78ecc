#!/usr/bin/env python
"""bench.py -- PPO optimizer-step throughput (OpenAI Five LSTM-4096, arXiv 1912.06680) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--B B]

One step = one pass of the whole hot path a1-a10 (GAE, TBPTT-16 forward through the
4096-unit LSTM + heads, PPO loss/grad, backward, DP gradient average, Adam with the
+-5 sqrt(v) clip) over one minibatch of B sequences per GPU.  Default
workload = BASELINE configs[1]: H=4096, D=4032, T=16, B=38,400 sequences per GPU
(= 7,680 paper samples of 5 hero replicas x 16 steps), weak scaling.
metric: paper samples/s (whole job); sequences/s and timesteps/s are reported beside it.

For N>1 launch with torchrun (one process per GPU, NCCL).  --impl reference times the
float64 oracle (the reference arm of this tier) on a bounded sample on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PPO train samples/s, LSTM-4096 16-step BPTT, 1/2/4/8 B200; % of roofline"
UNIT = "samples/s"
SEQ_PER_SAMPLE = 5   # a paper sample = 5 hero replicas x 16 steps


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--B", type=int, default=38400, help="sequences per GPU")
    ap.add_argument("--small-B", type=int, default=600,
                    help="--config paper-mb: sequences per GPU (default the paper's 600)")
    ap.add_argument("--H", type=int, default=4096)
    ap.add_argument("--D", type=int, default=4032)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alone", action="store_true",
                    help="skip the isolated loss/Adam kernel timings")
    ap.add_argument("--no-overlap", action="store_true",
                    help="fused DP exchange: do not overlap W_xh's exchange with the dW_o GEMM")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seq", type=int, default=1, help="oracle sample: sequences per step")
    ap.add_argument("--aux", action="store_true",
                    help="NEXT-4: with the aux heads (win, rank, 18 buildings) and their targets")
    ap.add_argument("--dx", action="store_true",
                    help="NEXT-4: also produce dL/dx for the observation network each step")
    ap.add_argument("--dp", choices=["nccl", "fused", "fused-push"], default="fused",
                    help="N>1 gradient exchange: nccl = ncclAvg allreduce + replicated Adam; "
                         "fused = one NVLink peer-memory kernel per rank (reduce-scatter of the "
                         "gradient shards, Adam on 1/N, all-gather of the bf16 shadow); "
                         "fused-push = the backward's epilogues push the shards to their owners")
    ap.add_argument("--infer-B", type=str, default="60,1,240,960",
                    help="--config infer: comma-separated batch sizes (first = headline)")
    ap.add_argument("--config", choices=["full", "gae", "iteration", "infer", "tiny", "paper-mb"],
                    default="full",
                    help="full: the PPO step (default); gae: GAE-only HBM sweep (configs[3]); "
                         "iteration: NEXT-1, steps drawn from a device experience buffer; "
                         "tiny: configs[0] (H=128, D=256, B=32) latency, eager and CUDA graph; "
                         "paper-mb: the paper's per-GPU minibatch (B=600, P:667), eager and graph")
    return ap.parse_args()


# ------------------------------------------------------------------ measured peaks
def peaks():
    p = {"hbm_gbs": 6551.0, "bf16_tflops": 1644.0, "bf16_tflops_sustained": 1362.1,
         "source": "MEASURED_PEAKS.json"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained"):
            if k in j:
                p[k] = float(j[k])
    except OSError:
        p.update(hbm_gbs=6650.0, bf16_tflops=1590.0, bf16_tflops_sustained=1400.0,
                 source="fallback (B200_PROFILING.md)")
    return p


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ oracle sample (CPU)
def oracle_sample_step(ctx):
    """One bounded sample of the step on the float64 oracle (test infrastructure): GAE over
    the sample's 256-step stream, TBPTT-16 forward/backward of `nseq` full-width sequences,
    PPO loss, and Adam over a 1/B share of the parameters (Adam runs once per B-sequence
    minibatch in the real step, so its per-sequence cost is 1/B of a full update)."""
    import numpy as np
    import oracle
    from oracle.step import loss_and_grads
    A, R = oracle.gae(ctx["ro"]["r"], ctx["ro"]["V"], ctx["ro"]["done"], ctx["gamma"], 0.95)
    T = ctx["cfg"].T
    adv = oracle.segments_to_sequences(A, T)[:, :ctx["nseq"]]
    ret = oracle.segments_to_sequences(R, T)[:, :ctx["nseq"]]
    _, g, _, _ = loss_and_grads(ctx["p"], ctx["seq"], ctx["logp_old"], adv, ret,
                                ctx["cfg"].head_sizes)
    share = ctx["adam_share"]
    for k in ("Wx", "Wh", "b", "Wo", "bo"):
        n = max(1, int(round(g[k].size * share)))
        p = ctx["p"][k].reshape(-1)[:n]
        z = np.zeros(n)
        oracle.adam_clip(p, g[k].reshape(-1)[:n], z, z, 1, 5e-5)


def oracle_context(H, D, nseq, B_full):
    import numpy as np
    import oracle
    import synth
    cfg = synth.Config(H=H, D=D, B=nseq)
    p = {k: v.astype(np.float64) for k, v in synth.make_params(cfg, 0).items()}
    seq = synth.make_sequences(cfg, 0)
    ro = synth.make_rollouts(1, 256, 0)
    logp_old = seq["logp_noise"].astype(np.float64) - 5.0
    return dict(cfg=cfg, p=p, seq=seq, ro=ro, logp_old=logp_old, nseq=nseq,
                gamma=oracle.gamma_from_horizon(180.0), adam_share=nseq / B_full)


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max((d.get("num_threads", 1) for d in info), default=os.cpu_count())
    except Exception:
        return os.cpu_count()


def run_reference(args):
    """--impl reference: the oracle as it stands, rank 0 only, bounded samples."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ctx = oracle_context(args.H, args.D, args.ref_seq, args.B)
    for _ in range(args.warmup):
        oracle_sample_step(ctx)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle_sample_step(ctx)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = (args.ref_seq / SEQ_PER_SAMPLE) / t
    sample = (f"{args.ref_seq} full-width sequence(s) (H={args.H}, D={args.D}, T=16) per step: "
              f"GAE + TBPTT fwd/bwd + loss + Adam on a {args.ref_seq}/{args.B} share of theta")
    cores = blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, n):
    return {
        "workload": (f"full OpenAI-Five LSTM-{args.H} PPO step: D={args.D}, T=16, "
                     f"B={args.B} sequences/GPU ({args.B // SEQ_PER_SAMPLE} paper samples), "
                     f"A={656 + (sum(__import__('synth').AUX_SIZES) if getattr(args, 'aux', False) else 0)}"
                     f" (7 factorised heads + value), GAE over 256-step segments"
                     + (", + dL/dx for the observation network" if getattr(args, "dx", False)
                        else "")
                     + (", + aux heads (win, rank, 18 buildings)" if getattr(args, "aux", False)
                        else "")),
        "H": args.H, "D": args.D, "T": 16, "B_per_gpu": args.B,
        "global_batch_samples": args.B * n // SEQ_PER_SAMPLE,
        "global_batch_timesteps": args.B * n * 16,
        "parallelism": f"dp{n}",
        "dp_exchange": (None if n == 1 else
                        "fused: NVLink peer-memory reduce-scatter + Adam on 1/N + bf16 all-gather"
                        + ("" if getattr(args, "no_overlap", False) else
                           "; W_xh's exchange overlapped with the dW_o GEMM")
                        if getattr(args, "dp", "nccl") == "fused" else
                        "fused-push: gradient shards pushed to their owners over NVLink from the "
                        "backward's epilogues + Adam on 1/N + bf16 all-gather"
                        if getattr(args, "dp", "nccl") == "fused-push"
                        else "NCCL allreduce (avg)"),
        "l2": "inputs larger than L2 (x alone is T*B*D*2 bytes per step)",
        "dx": bool(getattr(args, "dx", False)),
        "aux_heads": list(__import__("synth").AUX_SIZES) if getattr(args, "aux", False) else None,
    }


# ------------------------------------------------------------------ our arm
def algorithmic(H, D, T, B, A, nparam):
    """Algorithmic work per launch-class: flops for GEMMs, bytes for
    the HBM-bound kernels."""
    G4 = 4 * H
    rows = T * B
    return {
        "lstm_fwd_step": ("flop", 2.0 * B * G4 * (D + H) * T),
        "heads_fwd": ("flop", 2.0 * rows * A * H),
        "lstm_bwd_step": ("flop", 2.0 * B * H * G4 * (T - 1) + 2.0 * B * H * A * T),
        "wgrad_xh": ("flop", 2.0 * G4 * (D + H) * rows),
        "wgrad_o": ("flop", 2.0 * A * H * rows),
        "gae": ("byte", 17.0 * rows + 4.0 * rows / 256),
        "loss": ("byte", rows * (4.0 * A + 2.0 * A + 4 * 7 + 7 + 30 + 4 * 4 + 1)),
        "adam": ("byte", 30.0 * nparam),
        "pack_x": ("byte", rows * D * 2.0 + (T + 1) * B * (D + H + 64) * 2.0 + 8.0 * B * H),
        # h0, c0 in (fp32); h0 bf16 + c0 fp32 out; the [1 | 0...] pad of T+1 slots
        "pack_state": ("byte", 8.0 * B * H + 6.0 * B * H + (T + 1) * B * 64 * 2.0),
        "input_grad": ("flop", 2.0 * rows * G4 * D),
        # small-B backward (split-K dh GEMM + cell kernel): dh in, gates -> dz, c_t, c_{t-1},
        # dc in/out per step (the extra split partials are implementation traffic)
        "cell_bwd": ("byte", T * B * H * (4.0 + 2 * 8.0 + 4 * 4.0)),
    }


def run_gae_sweep(args):
    """BASELINE configs[3]: GAE over long rollouts (segment 256 ... a whole game, 10^6 steps),
    algorithmic 17 B/timestep (r, V, d in; A, R out) against the measured HBM peak."""
    import torch
    import synth
    from paper_1912_06680_b200 import _lib as L
    dev = torch.device("cuda", 0)
    pk = peaks()
    gamma = 1.0 - (4.0 / 30.0) / 180.0
    rows = []
    for steps in (10 ** 6, 10 ** 8, 10 ** 9):
        for Lr in (256, 1350, 6300, 20000, 10 ** 6):
            R = max(1, steps // Lr)
            n = R * Lr
            ro = synth.torch_rollouts(R, Lr, 1, dev)
            adv = torch.empty((R, Lr), device=dev)
            ret = torch.empty((R, Lr), device=dev)
            nb = L.gae_scratch_bytes(R, Lr)
            scratch = torch.empty(nb, dtype=torch.uint8, device=dev) if nb else None
            for _ in range(args.warmup):
                L.ppo_gae(ro["rew"], ro["val"], ro["done"], gamma, 0.95, adv, ret, scratch=scratch)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(args.steps):
                L.ppo_gae(ro["rew"], ro["val"], ro["done"], gamma, 0.95, adv, ret, scratch=scratch)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            gbs = 17.0 * n / (ms / 1e3) / 1e9
            rows.append({"L": Lr, "R": R, "timesteps": n, "ms": ms, "GB_s": gbs,
                         "frac": gbs / pk["hbm_gbs"], "timesteps_per_s": n / (ms / 1e3)})
            del ro, adv, ret, scratch
            torch.cuda.empty_cache()
    # NEXT-2: reward pipeline fused into GAE, 10 heroes per game, L = 256 segments
    rrows = []
    for steps in (10 ** 8, 10 ** 9):
        Lr = 256
        G = steps // (10 * Lr)
        n = G * 10 * Lr
        g = torch.Generator(device=dev).manual_seed(3)
        shaped = torch.randn((G, 10, Lr), generator=g, device=dev)
        win = torch.zeros((G, 10, Lr), device=dev)
        step0 = torch.randint(0, 20000, (G,), generator=g, device=dev, dtype=torch.int32)
        val = torch.randn((G * 10, Lr + 1), generator=g, device=dev)
        done = (torch.rand((G, Lr), generator=g, device=dev) < 1e-4).to(torch.uint8)
        adv = torch.empty((G * 10, Lr), device=dev)
        ret = torch.empty((G * 10, Lr), device=dev)
        stats = torch.zeros(3, dtype=torch.float64, device=dev)
        scratch = torch.empty(L.reward_gae_scratch_bytes(), dtype=torch.uint8, device=dev)
        cfg = L.ppo_reward_cfg(0.3, 0.6, 600.0, 4.0 / 30.0, 1)
        call = lambda: L.ppo_reward_gae(shaped, win, step0, val, done, cfg, stats, gamma, 0.95,
                                        adv, ret, scratch)
        for _ in range(args.warmup):
            call()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        # algorithmic: shaped, win, V in; A, R out (4 B each) + done (1 B per game-step)
        gbs = (20.0 * n + 1.0 * n / 10) / (ms / 1e3) / 1e9
        rrows.append({"kernel": "reward_gae", "L": Lr, "games": G, "hero_steps": n, "ms": ms,
                      "GB_s": gbs, "frac": gbs / pk["hbm_gbs"]})
        del shaped, win, step0, val, done, adv, ret
        torch.cuda.empty_cache()
    rows += rrows
    top = max((r for r in rows if r.get("timesteps", 0) >= 10 ** 9), key=lambda r: r["GB_s"])
    print(json.dumps({
        "metric": "GAE timesteps/s (configs[3] sweep)", "value": top["timesteps_per_s"],
        "unit": "timesteps/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "GAE-only, R streams x L steps, lambda 0.95, gamma(180 s)"},
        "roofline": {"bound": "hbm", "achieved": top["GB_s"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": top["frac"], "traffic": None, "kernel": "gae"},
        "sweep": rows}), flush=True)


def run_iteration(args):
    """NEXT-1: gradient steps sampled from a device-resident experience buffer (4x the
    minibatch), GAE at ingest, gather straight into the workspace, version publish every 32."""
    import torch
    import synth
    from paper_1912_06680_b200 import PPOOptimizer, _lib as L
    from paper_1912_06680_b200.trainer import ExperienceBuffer, PPOTrainer
    dev = torch.device("cuda", 0)
    H, D, T, B = args.H, args.D, 16, args.B
    cap = 4 * B
    cfg = synth.Config(H=H, D=D, B=B, T=T)
    opt = PPOOptimizer(D, H, B, T, cfg.head_sizes, precision="bf16", device=dev)
    prm = synth.torch_params(cfg, 0, dev)
    opt.load_canonical(prm["Wx"], prm["Wh"], prm["b"], prm["Wo"], prm["bo"])
    del prm
    buf = ExperienceBuffer(cap, D, H, T, cfg.head_sizes, bf16=True, device=dev)
    gamma = 1.0 - (4.0 / 30.0) / 180.0
    chunk = B  # push in chunks of B sequences (B/16 segments)
    for c in range(cap // chunk):
        sq = synth.torch_sequences(synth.Config(H=H, D=D, B=chunk, T=T), 100 + c, dev)
        ro = synth.torch_rollouts(chunk // 16, 256, 100 + c, dev)
        seg = dict(x=sq["x"].transpose(0, 1).contiguous(), h0=sq["h0"], c0=sq["c0"],
                   act=sq["act"].transpose(0, 1).contiguous(),
                   head_on=sq["head_on"].transpose(0, 1).contiguous(),
                   avail=sq["avail"].transpose(0, 1).contiguous(),
                   logp_old=(sq["logp_noise"] - 10.0).transpose(0, 1).contiguous(),
                   rew=ro["rew"], val=ro["val"], done=ro["done"])
        buf.push_segments(seg, gamma, 0.95)
        del sq, ro, seg
    torch.cuda.empty_cache()
    tr = PPOTrainer(opt, buf, seed=1)
    for _ in range(args.warmup):
        tr.step()
    torch.cuda.synchronize()
    L.prof_start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = max(args.steps, 1)
    for i in range(n):
        tr.step()
        if tr.global_step % 32 == 0:
            tr.published.copy_(opt.weights, non_blocking=True)
            tr.version += 1
    e1.record()
    torch.cuda.synchronize()
    prof = L.prof_stop()
    ms = e0.elapsed_time(e1) / n
    pk = peaks()
    gx = prof.get("gather_x", (0, 0.0))
    gr = prof.get("gather_rows", (0, 0.0))
    # gather: read x (T D 2 B) + h0/c0 (8 H) per sequence, write XH x-part + pads + h/c slots
    gbytes = B * (2.0 * T * D * 2 + 8 * H + 4 * H + 2 * H + (T + 1) * 128)
    g_ms = gx[1] / n
    print(json.dumps({
        "metric": "PPO train samples/s from the experience buffer (NEXT-1)",
        "value": B / 5 / (ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": n, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"B={B} sequences/step sampled with replacement from a "
                               f"{cap}-sequence device buffer (GAE at ingest)"},
        "gather": {"ms_per_step": g_ms, "rows_ms_per_step": gr[1] / n,
                   "achieved_GB_s": gbytes / (g_ms / 1e3) / 1e9 if g_ms else None,
                   "peak": pk["hbm_gbs"]},
        "kernels": {k: {"launches": c, "ms_per_step": t / n} for k, (c, t) in prof.items()},
        "sample_reuse": tr.sample_reuse}), flush=True)


def run_infer(args):
    """NEXT-3: forward-pass inference steps at the rollout batch (~60): one LSTM step +
    heads + masked sampling per call, state carried.  HBM-bound on the weights: algorithmic
    bytes per step = W_xh_aug + W_o_aug (bf16) + x + h/c read and written + outputs."""
    import torch
    import synth
    from paper_1912_06680_b200 import _lib as L
    from paper_1912_06680_b200.infer import PolicyServer
    dev = torch.device("cuda", 0)
    H, D = args.H, args.D
    pk = peaks()
    cfg0 = synth.Config(H=H, D=D, B=1, T=1)
    prm = synth.torch_params(cfg0, 0, dev)
    rows = []
    for B in [int(v) for v in args.infer_B.split(",")]:
        cfg = synth.Config(H=H, D=D, B=B, T=1)
        table = torch.from_numpy(synth.heads_on_table(cfg.head_sizes))
        srv = PolicyServer(D, H, B, cfg.head_sizes, device=dev, head_table=table, seed=3)
        theta = torch.empty(srv.layout.n_total, device=dev)
        L.ppo_pack_params(srv.dims, prm["Wx"], prm["Wh"], prm["b"], prm["Wo"], prm["bo"], theta)
        shadow = torch.empty(srv.layout.n_total, dtype=torch.bfloat16, device=dev)
        L.ppo_cast_bf16(theta, shadow)
        srv.load(shadow)
        del theta
        sq = synth.torch_sequences(synth.Config(H=H, D=D, B=B, T=16), 5, dev)
        xs = sq["x"]                      # [16][B][D] bf16: 16 distinct steps of input
        avail = sq["avail"]
        srv.reset(sq["h0"], sq["c0"])
        nsteps = max(args.steps, 16) * 8
        for i in range(args.warmup * 8):
            srv.step(xs[i % 16], avail[i % 16])
        torch.cuda.synchronize()
        L.prof_start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(nsteps):
            srv.step(xs[i % 16], avail[i % 16], want_out=False)
        e1.record()
        torch.cuda.synchronize()
        prof = L.prof_stop()
        us = e0.elapsed_time(e1) / nsteps * 1e3
        # CUDA graph of 16 consecutive steps (distinct inputs and counters), replayed
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            srv.step(xs[0], avail[0], want_out=False)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for i in range(16):
                    srv.step(xs[i], avail[i], want_out=False)
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        reps = max(1, nsteps // 16)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us_graph = e0.elapsed_time(e1) / (reps * 16) * 1e3
        # cuBLAS reference for the dominant GEMM (library baseline, same operands)
        lay = srv.layout
        Kx, G4 = D + H + 64, 4 * H
        wx = shadow[:G4 * Kx].view(G4, Kx)
        xh = torch.randn(B, Kx, device=dev).bfloat16()
        for _ in range(3):
            torch.matmul(xh, wx.t())
        torch.cuda.synchronize()
        e0.record()
        for _ in range(nsteps):
            torch.matmul(xh, wx.t())
        e1.record()
        torch.cuda.synchronize()
        us_cublas = e0.elapsed_time(e1) / nsteps * 1e3
        A, Ko = cfg.A, H + 64
        w_bytes = 2.0 * (G4 * Kx + A * Ko)
        io_bytes = B * (2.0 * D + 16.0 * H + 4 * 7 + 7 + 8 + A)
        step_bytes = w_bytes + io_bytes
        gates = prof.get("infer_gates", (1, 0.0))
        g_us = gates[1] / gates[0] * 1e3
        kern = {k: {"launches_per_step": c // nsteps, "us_per_step": t / nsteps * 1e3}
                for k, (c, t) in prof.items()}
        step_flop = 2.0 * B * (G4 * Kx + A * Ko)
        t_roof = max(step_bytes / (pk["hbm_gbs"] * 1e9),
                     step_flop / (pk["bf16_tflops_sustained"] * 1e12))
        rows.append({
            "B": B, "us_per_step": us, "us_per_step_graph": us_graph,
            # the bound flips from the weights' HBM stream to the tensor pipe as B grows
            "bound": "hbm" if step_bytes / (pk["hbm_gbs"] * 1e9) >= step_flop / (
                pk["bf16_tflops_sustained"] * 1e12) else "tensor",
            "roofline_frac": t_roof / (us_graph * 1e-6),
            "steps_per_s": 1e6 / us_graph, "hero_actions_per_s": B * 1e6 / us_graph,
            "achieved_GB_s": step_bytes / (us_graph * 1e-6) / 1e9,
            "frac": step_bytes / (us_graph * 1e-6) / 1e9 / pk["hbm_gbs"],
            "gates_gemm": {"us": g_us, "GB_s": 2.0 * G4 * Kx / (g_us * 1e-6) / 1e9,
                           "frac": 2.0 * G4 * Kx / (g_us * 1e-6) / 1e9 / pk["hbm_gbs"],
                           "cublas_us": us_cublas},
            "kernels": kern})
        del srv, sq, xs, avail, g, shadow, wx, xh
        torch.cuda.empty_cache()
    head = rows[0]
    print(json.dumps({
        "metric": "inference step latency (NEXT-3: LSTM step + heads + masked sampling)",
        "value": head["us_per_step_graph"], "unit": "us/step", "higher_is_better": False,
        "n_gpus": 1, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"forward-pass batch B={head['B']} (P:1263), H={H}, D={D}",
                   "l2": f"weights {2.0 * (4 * H * (D + H + 64)) / 1e6:.0f} MB > L2: streamed "
                         "from HBM every step"},
        "roofline": {"bound": "hbm", "achieved": head["achieved_GB_s"], "peak": pk["hbm_gbs"],
                     "unit": "GB/s", "frac": head["frac"], "kernel": "whole step (graph)"},
        "sweep": rows}), flush=True)


def run_small(args):
    """Latency-bound step configs on one GPU, timed eager and as one CUDA-graph replay per
    step (PPOOptimizer.capture): configs[0] tiny (H=128, D=256, 32 sequences) and the paper's
    own per-GPU minibatch (B = 600 sequences = 120 samples) at full width.  L2
    is flushed (a 256 MB write) between timed steps, outside the timed events."""
    import torch
    import synth
    from paper_1912_06680_b200 import PPOOptimizer, _lib as L
    dev = torch.device("cuda", 0)
    if args.config == "tiny":
        H, D, B = 128, 256, 32
    else:
        H, D, B = args.H, args.D, args.small_B
    T = 16
    cfg = synth.Config(H=H, D=D, B=B, T=T)
    opt = PPOOptimizer(D, H, B, T, cfg.head_sizes, precision="bf16", device=dev)
    prm = synth.torch_params(cfg, 0, dev)
    opt.load_canonical(prm["Wx"], prm["Wh"], prm["b"], prm["Wo"], prm["bo"])
    seq = synth.torch_sequences(cfg, 1000, dev)
    # rollout segments of 256 steps when B*T fills whole segments (tiny: 2 x 256);
    # B = 600 x 16 steps = 37.5 segments, so there 60 segments of 160 steps
    Lseg = 256 if (B * T) % 256 == 0 else 160
    ro = synth.torch_rollouts(B * T // Lseg, Lseg, 1000, dev)
    batch = dict(x=seq["x"], h0=seq["h0"], c0=seq["c0"], act=seq["act"], head_on=seq["head_on"],
                 avail=seq["avail"], rew=ro["rew"], val=ro["val"], done=ro["done"])
    batch["logp_old"] = opt.current_logp(batch) + seq["logp_noise"]
    opt.put_x(batch["x"])
    x_dev = batch.pop("x")
    opt.use_device_t()
    for _ in range(max(args.warmup, 1)):
        opt.step(batch)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def timed(fn, n):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(n)]
        for a, b in ev:
            flush.fill_(1)                       # L2 flush, outside the timed region
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in ev]

    clocks = Clocks(0)
    clocks.start()
    time.sleep(0.2)
    L.prof_start()
    eager = timed(lambda: opt.step(batch), args.steps)
    prof = L.prof_stop()
    graph = opt.capture(batch)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    replay = timed(graph.replay, args.steps)
    clk = clocks.stop()
    ms_e, ms_g = statistics.median(eager), statistics.median(replay)
    pk = peaks()
    alg = algorithmic(H, D, T, B, cfg.A, opt.layout.n_total)
    flop = sum(w for k, (kind, w) in alg.items() if kind == "flop" and k in prof)
    hbm = sum(w for k, (kind, w) in alg.items() if kind == "byte" and k in prof)
    t_roof = flop / (pk["bf16_tflops_sustained"] * 1e12) + hbm / (pk["hbm_gbs"] * 1e9)
    kernels = {k: {"launches_per_step": n // args.steps, "us_per_step": t / args.steps * 1e3}
               for k, (n, t) in prof.items()}
    n_launch = sum(n for n, _ in prof.values())
    # end to end: inputs from pinned host memory each step (x into the workspace), stats back
    keys = ("h0", "c0", "rew", "val", "done", "act", "head_on", "avail", "logp_old")
    host = {k: batch[k].cpu().pin_memory() for k in keys}
    host_x = x_dev.cpu().pin_memory()
    st_host = torch.empty(8, dtype=torch.float32).pin_memory()
    h2d = sum(v.numel() * v.element_size() for v in host.values()) + \
        host_x.numel() * host_x.element_size()

    def e2e_step():
        for k in keys:
            batch[k].copy_(host[k], non_blocking=True)
        opt.put_x(host_x)
        graph.replay()
        st_host.copy_(opt.stats[:8], non_blocking=True)
    e2e = timed(e2e_step, args.steps)
    ms_x = statistics.median(e2e)
    tiny = args.config == "tiny"
    line = {
        "metric": ("PPO step latency, tiny config (configs[0])" if tiny else
                   "PPO train samples/s at the paper's per-GPU minibatch (B=600, P:667)"),
        "value": ms_g * 1e3 if tiny else B / (ms_g / 1e3) / SEQ_PER_SAMPLE,
        "unit": "us/step" if tiny else UNIT, "higher_is_better": not tiny,
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_g,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded; paper-shaped rollouts, random-init weights)",
        "config": {"workload": (f"{'tiny' if tiny else 'paper minibatch'} PPO step: H={H}, D={D}, "
                                f"T=16, B={B} sequences ({B // SEQ_PER_SAMPLE} paper samples), "
                                f"GAE over {Lseg}-step segments + TBPTT fwd/bwd + loss + Adam"),
                   "H": H, "D": D, "T": T, "B_per_gpu": B, "parallelism": "dp1",
                   "l2": "flushed between timed steps (256 MB write outside the timed events)",
                   "timing": "median of per-step CUDA events; value from the CUDA-graph replay"},
        "eager": {"ms_per_step": ms_e, "samples_per_s": B / (ms_e / 1e3) / SEQ_PER_SAMPLE},
        "graph": {"ms_per_step": ms_g, "samples_per_s": B / (ms_g / 1e3) / SEQ_PER_SAMPLE},
        "roofline": {"bound": "tensor", "kernel": "whole step (graph replay)",
                     "achieved": flop / (ms_g / 1e3) / 1e12, "unit": "TFLOP/s",
                     "peak": pk["bf16_tflops_sustained"],
                     "frac": flop / (ms_g / 1e3) / 1e12 / pk["bf16_tflops_sustained"],
                     "traffic": None, "step": {"T_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms_g,
                                               "flop": flop, "hbm_bytes": hbm}},
        "e2e": {"value": ms_x * 1e3 if tiny else B / (ms_x / 1e3) / SEQ_PER_SAMPLE,
                "unit": "us/step" if tiny else UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": st_host.numel() * 4, "ms_per_step": ms_x,
                "note": "inputs copied from pinned host memory, then the graph replay, then the "
                        "stats read back, all inside the timed events"},
        "cpu_baseline": None, "gpu_launches": n_launch, "clocks": clk, "kernels": kernels,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.config in ("tiny", "paper-mb"):
        run_small(args)
        return
    if args.config == "infer":
        run_infer(args)
        return
    if args.config == "iteration":
        run_iteration(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    if args.config == "gae":
        run_gae_sweep(args)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)

    import synth
    from paper_1912_06680_b200 import PPOOptimizer, _lib as L

    from paper_1912_06680_b200 import dist as pdist
    comm = pdist.make_comm(device)

    H, D, T, B = args.H, args.D, 16, args.B
    aux = synth.AUX_SIZES if args.aux else (0, 0, 0)
    cfg = synth.Config(H=H, D=D, B=B, T=T, aux=aux)
    mk = lambda dp: PPOOptimizer(D, H, B, T, cfg.head_sizes, precision="bf16",  # noqa: E731
                                 device=device, comm=comm, n_buckets=8,
                                 n_ws=1 if args.no_e2e else 2, aux=aux, dp=dp,
                                 overlap=not args.no_overlap)
    opt = None
    if comm is not None and args.dp.startswith("fused"):
        # the peer mappings (CUDA IPC) need plain cudaMalloc'd buffers; every rank must agree
        # before the first collective step, else all fall back to the NCCL allreduce
        try:
            opt, ok = mk(args.dp), 1.0
        except L.PPOError as e:
            ok = 0.0
            print(f"[bench] fused DP exchange unavailable on rank {rank}: {e}", file=sys.stderr)
        if -pdist.max_over_ranks(-ok, device) < 1.0:
            opt, args.dp = None, "nccl"
    if opt is None:
        opt = mk("allreduce")
    prm = synth.torch_params(cfg, 0, device)          # same init on every rank
    opt.load_canonical(prm["Wx"], prm["Wh"], prm["b"], prm["Wo"], prm["bo"])
    del prm
    seq = synth.torch_sequences(cfg, 1000 + rank, device)
    R = B * T // 256
    ro = synth.torch_rollouts(R, 256, 1000 + rank, device)
    batch = dict(x=seq["x"], h0=seq["h0"], c0=seq["c0"], act=seq["act"],
                 head_on=seq["head_on"], avail=seq["avail"], rew=ro["rew"], val=ro["val"],
                 done=ro["done"])
    if args.aux:
        batch.update(synth.torch_aux(R, 256, aux, 1000 + rank, device))
    # behaviour log-probs = current policy + N(0, 0.1^2) (forward-pass GPUs)
    batch["logp_old"] = opt.current_logp(batch) + seq["logp_noise"]
    # the resident batch's x lives in the workspace's x rows (zero-copy, ppo_copy_x): the step
    # packs only h0/c0 into the recurrent slots
    opt.put_x(batch["x"])
    x_dev = batch.pop("x")
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    dx = torch.empty(T, B, D, device=device) if args.dx else None
    for _ in range(args.warmup):
        opt.step(batch, dx=dx)
    torch.cuda.synchronize()
    stats = opt.stats[:L.PPO_STATS].cpu().tolist()

    clocks = Clocks(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    L.prof_start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        opt.step(batch, dx=dx)
    e1.record(stream)
    torch.cuda.synchronize()
    prof = L.prof_stop()
    barrier()
    clk = clocks.stop()
    ms = pdist.max_over_ranks(e0.elapsed_time(e1), device)
    ms_step = ms / args.steps
    seq_s = B * world / (ms_step / 1e3)
    value = seq_s / SEQ_PER_SAMPLE

    # ---- roofline of each kernel class, dominant one reported
    pk = peaks()
    alg = algorithmic(H, D, T, B, cfg.A, opt.layout.n_total)
    kernels = {}
    for tag, (n, tot) in prof.items():
        per_step_ms = tot / args.steps
        ent = {"launches_per_step": n // args.steps, "ms_per_step": per_step_ms,
               "share": per_step_ms / ms_step}
        if tag in alg:
            kind, work = alg[tag]
            if kind == "flop":
                ach = work / (per_step_ms / 1e3) / 1e12
                ent.update(bound="tensor", achieved=ach, unit="TFLOP/s",
                           peak=pk["bf16_tflops_sustained"], frac=ach / pk["bf16_tflops_sustained"])
            else:
                ach = work / (per_step_ms / 1e3) / 1e9
                ent.update(bound="hbm", achieved=ach, unit="GB/s", peak=pk["hbm_gbs"],
                           frac=ach / pk["hbm_gbs"])
        kernels[tag] = ent
    # DRAM traffic per launch from the committed ncu --set full capture of this config
    traffic, traffic_src = {}, None
    for name in ("r02_traffic.json", "r01_traffic.json"):   # the newest capture present
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                traffic = json.load(f)["kernels"]
            traffic_src = f"profiles/{name} (ncu --set full, B=38400)"
            break
        except (OSError, KeyError, ValueError):
            pass
    for tag, ent in kernels.items():
        if tag in traffic:
            ent["traffic_per_launch"] = traffic[tag]["dram_bytes_per_launch"]
    dom = max((k for k in kernels if "achieved" in kernels[k]),
              key=lambda k: kernels[k]["ms_per_step"])
    d = kernels[dom]
    n_launch = sum(n for n, _ in prof.values())
    step_flop = sum(w for k, (kind, w) in alg.items() if kind == "flop" and k in prof)
    roofline = {"bound": d["bound"], "achieved": d["achieved"], "peak": d["peak"],
                "unit": d["unit"], "frac": d["frac"],
                "traffic": traffic.get(dom, {}).get("dram_bytes_per_launch") if B == 38400 else None,
                "traffic_source": traffic_src,
                "kernel": dom, "launches_per_step": d["launches_per_step"],
                "peak_source": pk["source"] + (" sustained" if d["bound"] == "tensor" else ""),
                "step_tflops": step_flop / (ms_step / 1e3) / 1e12,
                "step_frac_of_sustained_bf16": step_flop / (ms_step / 1e3) / 1e12 / pk["bf16_tflops_sustained"]}
    # whole-step roofline: every GEMM at the sustained bf16 peak plus every
    # HBM-bound kernel at the measured HBM bandwidth, against the measured step time
    step_bytes = sum(w for k, (kind, w) in alg.items() if kind == "byte" and k in prof)
    t_roof = step_flop / (pk["bf16_tflops_sustained"] * 1e12) + step_bytes / (pk["hbm_gbs"] * 1e9)
    roofline["step"] = {"T_roof_ms": t_roof * 1e3, "ms_per_step": ms_step,
                        "frac": t_roof * 1e3 / ms_step,
                        "flop": step_flop, "hbm_bytes": step_bytes}

    # ---- the HBM-bound kernels alone (informational, outside the timed region): each run
    # between 256 MB L2-flushing writes, at the clock a lone kernel gets; inside the step the
    # 1 kW power cap holds the SM clock near 1.2 GHz, which an issue-bound kernel (the loss)
    # feels and a bandwidth-bound one (Adam) hardly does
    if world == 1 and not getattr(args, "no_alone", False):
        flush = torch.empty(64 << 20, dtype=torch.float32, device=device)
        for tag, fn in (("loss", lambda: opt.loss(batch)), ("adam", lambda: opt.apply())):
            if tag not in kernels or "achieved" not in kernels[tag]:
                continue
            times = []
            for _ in range(7):
                flush.zero_()
                a0 = torch.cuda.Event(enable_timing=True)
                a1 = torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                fn()
                a1.record(stream)
                torch.cuda.synchronize()
                times.append(a0.elapsed_time(a1))
            t_ms = sorted(times)[len(times) // 2]
            kind, work = alg[tag]
            ach = work / (t_ms / 1e3) / 1e9
            kernels[tag]["alone"] = {"ms": t_ms, "achieved": ach, "unit": "GB/s",
                                     "frac": ach / pk["hbm_gbs"],
                                     "note": "median of 7 isolated launches, L2 flushed before "
                                             "each, outside the timed steps"}
        del flush

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # End to end through the public API with HOST inputs: every step's inputs are copied
        # from pinned host memory (H2D) and its stats read back (D2H) inside the timed region.
        # Inputs are double-buffered on the device: the H2D of step k+1 runs on a copy stream
        # while step k computes (the first step's copy overlaps only its own forward).
        # x goes straight from pinned host memory into the x rows of one of two workspaces,
        # one time slice at a time (ppo_copy_x_slice), and the forward's step t waits only for
        # slice t (lstm_bptt_fwd_ev); GAE's and the state's inputs go first, the loss's last.
        # The other inputs are double-buffered device tensors.
        keys_first = ("h0", "c0", "rew", "val", "done") + \
            (("last", "outcome", "rank", "events", "boot") if args.aux else ())
        keys_rest = ("act", "head_on", "avail", "logp_old")
        keys = keys_first + keys_rest
        host = {k: batch[k].cpu().pin_memory() for k in keys}
        host_x = x_dev.cpu().pin_memory()
        del x_dev
        h2d = sum(v.numel() * v.element_size() for v in host.values()) + \
            host_x.numel() * host_x.element_size()
        bufs = [{k: batch[k] for k in keys}, {k: torch.empty_like(batch[k]) for k in keys}]
        st_host = torch.empty(8, dtype=torch.float32).pin_memory()
        d2h = st_host.numel() * 4
        copy_stream = torch.cuda.Stream(device=device)
        ev_first = [torch.cuda.Event(), torch.cuda.Event()]
        ev_x = [[torch.cuda.Event() for _ in range(T)] for _ in range(2)]
        ev_rest = [torch.cuda.Event(), torch.cuda.Event()]
        used = [torch.cuda.Event(), torch.cuda.Event()]

        def upload(slot):
            copy_stream.wait_event(used[slot])
            with torch.cuda.stream(copy_stream):
                for k in keys_first:
                    bufs[slot][k].copy_(host[k], non_blocking=True)
                ev_first[slot].record(copy_stream)
                for t in range(T):
                    L.ppo_copy_x_slice(opt.dims, B, t, host_x[t], opt.ws_list[slot], copy_stream)
                    ev_x[slot][t].record(copy_stream)
                for k in keys_rest:
                    bufs[slot][k].copy_(host[k], non_blocking=True)
                ev_rest[slot].record(copy_stream)

        def run(nsteps):
            upload(0)
            for i in range(nsteps):
                cur = i % 2
                if i + 1 < nsteps:
                    upload(1 - cur)
                stream.wait_event(ev_first[cur])
                opt.select_ws(cur)
                opt.step_streamed(bufs[cur], ev_x[cur], ev_rest[cur], dx=dx)
                used[cur].record(stream)
                st_host.copy_(opt.stats[:8], non_blocking=True)

        run(2)
        torch.cuda.synchronize()
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        run(args.steps)
        f1.record(stream)
        torch.cuda.synchronize()
        ems = pdist.max_over_ranks(f0.elapsed_time(f1), device)
        e2e = {"value": B * world / (ems / args.steps / 1e3) / SEQ_PER_SAMPLE, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": ems / args.steps,
               "overlap": "H2D of step k+1 on a copy stream during step k (double-buffered "
                          "inputs; x straight into the workspace of step k+1, one time slice "
                          "at a time; step t of the forward waits only for slice t)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ctx = oracle_context(H, D, args.ref_seq, B)
        t0 = time.perf_counter()
        oracle_sample_step(ctx)
        tcpu = time.perf_counter() - t0
        cpu = {"value": (args.ref_seq / SEQ_PER_SAMPLE) / tcpu, "unit": UNIT,
               "cores": blas_threads(), "kind": "oracle",
               "sample": (f"{args.ref_seq} full-width sequence(s) per step: GAE + TBPTT-16 "
                          f"fwd/bwd + loss + Adam on a {args.ref_seq}/{B} share of theta; "
                          f"{tcpu:.1f} s")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (seeded; paper-shaped rollouts, random-init weights)",
            "config": workload_config(args, world),
            "sequences_per_s": seq_s, "timesteps_per_s": seq_s * T,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": n_launch, "clocks": clk, "kernels": kernels,
            "loss_stats_warmup": dict(zip(L.STAT_NAMES, stats)),
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        L.comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
