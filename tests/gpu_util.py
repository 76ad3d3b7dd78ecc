"""Helpers for the GPU parity tests: move seeded synth inputs to the device, run the oracle on
the same inputs, compare with the tolerances of DESIGN.md "Parity"."""
import numpy as np
import torch

import oracle
import synth
from oracle.step import loss_and_grads

HYPER = synth.HYPER


def elementwise_ok(x, ref, tol):
    """|x - ref| <= tol * (|ref| + rms(ref)) elementwise (north_star: GAE/loss 1e-5 rel)."""
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    rms = np.sqrt(np.mean(ref * ref)) if ref.size else 0.0
    bad = np.abs(x - ref) > tol * (np.abs(ref) + rms)
    return (not bad.any()), (np.abs(x - ref) / (np.abs(ref) + rms + 1e-300)).max() if ref.size else 0.0


def normwise(x, ref):
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    return np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-300)


def dev(a, device="cuda", dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a)).to(device)
    return t if dtype is None else t.to(dtype)


AUX_HYPER = dict(c_win=1.0, c_rank=1.0, c_bld=1.0, aux_win_trunk=0.01)


def aux_case(cfg, R, L, seed, hyper):
    """NEXT-4 inputs of R segments + the oracle's labels in minibatch layout [T][B][n_aux]
    (gamma2 fp32-rounded on both sides, like gamma in DESIGN Q18)."""
    from oracle.aux import aux_labels
    n_win, n_rank, n_bld = cfg.aux
    ax = synth.make_aux(R, L, cfg.aux, seed, p_last=0.3, p_event=0.02)
    g2 = float(np.float32(oracle.gamma_from_horizon(120.0, HYPER["T_step"])))
    lab = aux_labels(ax["last"].astype(bool), ax["outcome"], ax["rank"], ax["events"],
                     ax["boot"], g2, n_win, n_rank, n_bld)                 # [R][L][n_aux]
    n_aux = lab.shape[2]
    per = L // cfg.T
    # sequence b = r*per + l//T, step t = l % T  (the GAE minibatch mapping, DESIGN O3)
    mb = lab.reshape(R, per, cfg.T, n_aux).transpose(2, 0, 1, 3).reshape(cfg.T, R * per, n_aux)
    aux = dict(labels=mb, n_win=n_win, n_rank=n_rank, n_bld=n_bld, c_win=hyper["c_win"],
               c_rank=hyper["c_rank"], c_bld=hyper["c_bld"], win_trunk=hyper["aux_win_trunk"])
    return ax, g2, lab, aux


def make_case(cfg, seed, pad_frac=0.0, bo_scale=0.05, wo_scale=1.0, aux_hyper=None):
    """Seeded params/sequences/rollouts + oracle reference of one full step."""
    params = synth.make_params(cfg, seed, bo_scale=bo_scale)
    params["Wo"] = (params["Wo"] * wo_scale).astype(np.float32)
    seq = synth.make_sequences(cfg, seed, pad_frac=pad_frac)
    L = HYPER["segment"]
    assert (cfg.B * cfg.T) % L == 0
    R = cfg.B * cfg.T // L
    ro = synth.make_rollouts(R, L, seed, p_done=0.01)
    gamma = oracle.gamma_from_horizon(HYPER["horizon_s"], HYPER["T_step"])
    # both sides use the fp32-rounded gamma/lambda (DESIGN O1)
    gamma32, lam32 = float(np.float32(gamma)), float(np.float32(HYPER["lam"]))
    A, R_ = oracle.gae(ro["r"], ro["V"], ro["done"], gamma32, lam32)
    adv = oracle.segments_to_sequences(A, cfg.T)
    ret = oracle.segments_to_sequences(R_, cfg.T)
    p64 = {k: v.astype(np.float64) for k, v in params.items()}
    lp = loss_and_grads(p64, seq, np.zeros((cfg.T, cfg.B)), adv, ret, cfg.head_sizes)[3]["logpi"]
    logp_old = (lp.reshape(cfg.T, cfg.B) + seq["logp_noise"]).astype(np.float32)
    aux = None
    if sum(cfg.aux):
        _, _, _, aux = aux_case(cfg, R, L, seed, aux_hyper or AUX_HYPER)
    Lval, grads, stats, inter = loss_and_grads(p64, seq, logp_old.astype(np.float64), adv, ret,
                                               cfg.head_sizes, HYPER["clip_eps"], HYPER["c_v"],
                                               HYPER["c_e"], aux=aux)
    return dict(params=params, seq=seq, ro=ro, adv=adv, ret=ret, logp_old=logp_old, loss=Lval,
                grads=grads, stats=stats, inter=inter, gamma32=gamma32, aux=aux)


def device_batch(case, bf16, device="cuda"):
    s = case["seq"]
    ro = case["ro"]
    b = dict(
        x=dev(s["x"], device, torch.bfloat16 if bf16 else torch.float32),
        h0=dev(s["h0"], device), c0=dev(s["c0"], device),
        act=dev(s["act"], device), head_on=dev(s["head_on"], device),
        avail=dev(s["avail"], device), valid=dev(s["valid"], device),
        logp_old=dev(case["logp_old"], device),
        rew=dev(ro["r"], device), val=dev(ro["V"], device), done=dev(ro["done"], device),
    )
    if case.get("aux") is not None:
        b["aux_label"] = dev(case["aux"]["labels"].astype(np.float32), device)
    return b


def load_params(opt, params, device="cuda"):
    opt.load_canonical(*(dev(params[k], device) for k in ("Wx", "Wh", "b", "Wo", "bo")))
