"""ORACLE (test infrastructure only) -- one PPO optimizer step, composed in the paper's order.

P:1249-1255 [§3.2]: each optimizer GPU computes gradients on a minibatch, gradients are
averaged across the pool with allreduce "before being synchronously applied", then Adam
with the +-5 sqrt(v) clip.  Composition: GAE -> minibatch -> LSTM
forward (TBPTT-16) -> heads -> PPO loss -> backward -> DP average -> Adam.
"""
import numpy as np

from .adam import adam_clip
from .aux import aux_loss, trunk_gradient
from .gae import gae, segments_to_sequences
from .loss import heads_backward, heads_forward, ppo_loss
from .lstm import lstm_backward, lstm_forward

PARAM_NAMES = ("Wx", "Wh", "b", "Wo", "bo")


def loss_and_grads(params, seq, logp_old, adv, ret, head_sizes, clip_eps=0.2, c_v=1.0,
                   c_e=0.01, denom=None, aux=None):
    """Forward + loss + truncated BPTT on one shard.  seq: x [T][B][D], h0, c0 [B][H],
    act [T][B][nh], head_on, avail, valid [T][B]; logp_old/adv/ret [T][B].
    aux (NEXT-4, oracle/aux.py): dict labels [T][B][n_aux], n_win, n_rank, n_bld, c_win,
    c_rank, c_bld, win_trunk -- W_o/b_o then carry the aux rows after the value.
    Returns (L, grads dict, stats, intermediates)."""
    cache = lstm_forward(params["Wx"], params["Wh"], params["b"], seq["x"], seq["h0"], seq["c0"])
    T, B, H = cache["h"].shape
    hflat = cache["h"].reshape(T * B, H)
    Y = heads_forward(hflat, params["Wo"], params["bo"])
    A0 = sum(head_sizes) + 1
    L, dY0, stats, logpi = ppo_loss(Y[:, :A0], seq["act"], seq["head_on"], seq["avail"],
                                    logp_old, adv, ret, seq.get("valid"), head_sizes, clip_eps,
                                    c_v, c_e, denom)
    dY = np.zeros_like(Y)
    dY[:, :A0] = dY0
    dY_trunk = dY.copy()
    if aux is not None:
        n_aux = aux["n_win"] + aux["n_rank"] + aux["n_bld"]
        assert Y.shape[1] == A0 + n_aux
        La, dYa, comps = aux_loss(Y[:, A0:], np.asarray(aux["labels"]).reshape(T * B, n_aux),
                                  None if seq.get("valid") is None else
                                  np.asarray(seq["valid"]).reshape(-1),
                                  aux["n_win"], aux["n_rank"], aux["n_bld"], aux["c_win"],
                                  aux["c_rank"], aux["c_bld"], denom)
        L = L + La                                             # Q25: L = L_ppo + L_aux
        stats = dict(stats, loss_ppo=stats["loss"], loss=L, aux=La,
                     **{"aux_" + k: v for k, v in comps.items()})
        dY[:, A0:] = dYa                                        # the heads' own weights
        dY_trunk[:, A0:] = trunk_gradient(dYa, aux["n_win"], aux["win_trunk"])   # Q26
    dWo, dbo = heads_backward(hflat, dY)
    dh_out = (dY_trunk @ np.asarray(params["Wo"], np.float64)).reshape(T, B, H)
    dWx, dWh, db, dz = lstm_backward(cache, dh_out)
    grads = dict(Wx=dWx, Wh=dWh, b=db, Wo=dWo, bo=dbo)
    return L, grads, stats, dict(Y=Y, dY=dY, logpi=logpi, h=cache["h"], c=cache["c"], dz=dz)


def dp_average(shard_grads):
    """DESIGN O9: g = (1/N) sum_n g_n, then applied synchronously."""
    n = len(shard_grads)
    return {k: sum(g[k] for g in shard_grads) / n for k in shard_grads[0]}


def ppo_step(params, adam_state, seq, rollouts, logp_old, cfg, t):
    """One full optimizer step on one shard (N = 1).

    rollouts: r [R][L], V [R][L+1], done [R][L]; the minibatch sequences are the
    T-step windows of these streams (DESIGN O3).  cfg: gamma, lam, clip_eps, c_v, c_e,
    lr, beta1, beta2, adam_eps, clip_sigma, head_sizes.  adam_state: dict name ->
    (m, v).  Returns (new params, new adam_state, record)."""
    A, R = gae(rollouts["r"], rollouts["V"], rollouts["done"], cfg["gamma"], cfg["lam"])
    T = seq["x"].shape[0]
    adv = segments_to_sequences(A, T)
    ret = segments_to_sequences(R, T)
    L, grads, stats, inter = loss_and_grads(params, seq, logp_old, adv, ret, cfg["head_sizes"],
                                            cfg["clip_eps"], cfg["c_v"], cfg["c_e"])
    new_params, new_state = {}, {}
    for k in PARAM_NAMES:
        m, v = adam_state[k]
        new_params[k], m2, v2 = adam_clip(params[k], grads[k], m, v, t, cfg["lr"], cfg["beta1"],
                                          cfg["beta2"], cfg["adam_eps"], cfg["clip_sigma"])
        new_state[k] = (m2, v2)
    rec = dict(adv=adv, ret=ret, loss=L, grads=grads, stats=stats, **inter)
    return new_params, new_state, rec
