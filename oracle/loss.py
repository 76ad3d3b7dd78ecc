"""ORACLE (test infrastructure only) -- heads and the PPO clipped-surrogate loss.

P:618-619 [App. NN arch] "the value function is computed as another linear projection
of the LSTM state"; P:606 action logits are linear projections of the LSTM output.
P:1243 [§3.2] PPO [schulman2017proximal]; P:914 PPO clipping 0.2; P:915 value loss
weight 1.0; P:399-403 [App. Exploration] entropy bonus c S[pi](s_t), c = 0.01;
P:306 action filters restrict the primary action; P:308 ignored parameter heads are
masked out when optimizing; P:350-368 Table target types.

Row layout: rows are (t, b) flattened time-major (row = t*B + b).  Head outputs
y = [logits of 7 heads (DESIGN Q7 order) | value].
"""
import numpy as np

STAT_NAMES = ("loss", "pg", "vf", "ent", "approx_kl", "clipfrac", "n_valid", "flags")
FLAG_NONFINITE = 1
FLAG_ACTION_UNAVAILABLE = 2
FLAG_EMPTY_AVAIL = 4


def heads_forward(h, Wo, bo):
    """DESIGN O5: y = h W_o^T + b_o.  h [..][H] -> y [..][A]."""
    return np.asarray(h, np.float64) @ np.asarray(Wo, np.float64).T + np.asarray(bo, np.float64)


def heads_backward(h, dY):
    """Gradients of y = h W_o^T + b_o: dW_o = dY^T h, db_o = sum dY, dh = dY W_o
    (the last is returned by the caller, which owns W_o).  h [N][H], dY [N][A]."""
    h = np.asarray(h, np.float64)
    dY = np.asarray(dY, np.float64)
    return dY.T @ h, dY.sum(axis=0)


def _masked_log_softmax(logits, mask):
    """log softmax over entries with mask=1; masked entries get -inf."""
    z = np.where(mask, logits, -np.inf)
    m = np.max(z, axis=-1, keepdims=True)
    m = np.where(np.isfinite(m), m, 0.0)
    s = np.sum(np.where(mask, np.exp(z - m), 0.0), axis=-1, keepdims=True)
    return z - m - np.log(s)


def ppo_loss(Y, act, head_on, avail, logp_old, adv, ret, valid, head_sizes,
             clip_eps=0.2, c_v=1.0, c_e=0.01, denom=None):
    """DESIGN O6 (loss) and O7 (its analytic gradient).

    Per row with weight w = valid:
      lp_k    = log_softmax(l_k)   (primary: unavailable entries -> -inf)
      logpi   = sum_k on_k lp_k[a_k]              (masked heads)
      S       = sum_k on_k H(p_k), 0 log 0 = 0    (DESIGN Q7)
      rho     = exp(logpi - logpi_old)
      l_row   = -min(rho A, clip(rho, 1-eps, 1+eps) A) + c_v (V - R)^2 - c_e S
      L       = sum_rows w l_row / denom          (denom = rows, DESIGN Q9)
    Gradient (DESIGN Q8: unclipped branch carries gradient, ties included):
      g_pi    = -A rho [rho A <= clip(rho) A] w / denom
      dl_k    = on_k (g_pi (onehot(a_k) - p_k) + (c_e w / denom) p_k (log p_k + S_k))
      dV      = 2 c_v (V - R) w / denom
    Returns (L, dY [N][A], stats dict, logpi [N]).
    """
    Y = np.asarray(Y, np.float64)
    N, A = Y.shape
    nh = len(head_sizes)
    assert A == sum(head_sizes) + 1
    act = np.asarray(act).reshape(N, nh)
    head_on = np.asarray(head_on).reshape(N, nh).astype(np.float64)
    avail = np.asarray(avail).reshape(N, head_sizes[0]).astype(bool)
    logp_old = np.asarray(logp_old, np.float64).reshape(N)
    adv = np.asarray(adv, np.float64).reshape(N)
    ret = np.asarray(ret, np.float64).reshape(N)
    w = np.ones(N) if valid is None else np.asarray(valid, np.float64).reshape(N)
    if denom is None:
        denom = float(N)
    rows = np.arange(N)

    offs = np.concatenate([[0], np.cumsum(head_sizes)])
    logpi = np.zeros(N)
    ent = np.zeros(N)
    probs, logps, ents = [], [], []
    flags = 0
    for k in range(nh):
        lk = Y[:, offs[k]:offs[k + 1]]
        mask = avail if k == 0 else np.ones_like(lk, dtype=bool)
        lp = _masked_log_softmax(lk, mask)
        p = np.where(mask, np.exp(lp), 0.0)
        plogp = np.where(mask, p * np.where(mask, lp, 0.0), 0.0)
        Hk = -plogp.sum(axis=1)
        logpi += head_on[:, k] * lp[rows, act[:, k]]
        ent += head_on[:, k] * Hk
        probs.append(p)
        logps.append(lp)
        ents.append(Hk)
    if np.any(~avail[rows, act[:, 0]] & (w > 0)):
        flags |= FLAG_ACTION_UNAVAILABLE
    if np.any(~avail.any(axis=1) & (w > 0)):
        flags |= FLAG_EMPTY_AVAIL

    V = Y[:, A - 1]
    rho = np.exp(logpi - logp_old)
    surr1 = rho * adv
    surr2 = np.clip(rho, 1.0 - clip_eps, 1.0 + clip_eps) * adv
    unclipped = surr1 <= surr2
    pg_row = -np.minimum(surr1, surr2)
    vf_row = (V - ret) ** 2
    l_row = pg_row + c_v * vf_row - c_e * ent
    if not np.all(np.isfinite(l_row[w > 0])):
        flags |= FLAG_NONFINITE
    L = np.sum(w * l_row) / denom

    g_pi = -adv * rho * unclipped * w / denom
    ce = c_e * w / denom
    dY = np.zeros((N, A))
    for k in range(nh):
        p, lp, Hk = probs[k], logps[k], ents[k]
        onehot = np.zeros_like(p)
        onehot[rows, act[:, k]] = 1.0
        ent_term = np.where(p > 0, p * (np.where(p > 0, lp, 0.0) + Hk[:, None]), 0.0)
        dY[:, offs[k]:offs[k + 1]] = head_on[:, k:k + 1] * (
            g_pi[:, None] * (onehot - p) + ce[:, None] * ent_term)
    dY[:, A - 1] = 2.0 * c_v * (V - ret) * w / denom

    stats = dict(
        loss=L,
        pg=np.sum(w * pg_row) / denom,
        vf=np.sum(w * vf_row) / denom,
        ent=np.sum(w * ent) / denom,
        approx_kl=np.sum(w * (logp_old - logpi)) / denom,
        clipfrac=np.sum(w * (~unclipped)) / denom,
        n_valid=np.sum(w),
        flags=flags,
    )
    return L, dY, stats, logpi
