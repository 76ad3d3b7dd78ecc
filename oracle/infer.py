"""ORACLE (test infrastructure only) -- NEXT-3: one forward-pass inference step.

P:1263 [§3.2] the rollout machines "communicate with a separate pool of GPU machines which
run forward passes in larger batches of approximately 60": one policy step for a batch of
heroes = one LSTM step from each hero's carried state, the linear heads
(P:606), and a sample of the factorised action (P:303-368 [App. Action Space]):
the primary action restricted to the available ones (action filters), every
parameter head sampled, the heads the primary's target type reads (Table target types,
P:350-368) recorded, and the behaviour log-probability of the read heads (the logp_old the
optimizer's PPO ratio divides by).

Reading Q22: sampling is exact sampling from the softmax at temperature 1 by
the Gumbel-max rule  a = argmax_k (l_k + g_k),  g_k = -log(-log u_k),  ties -> smallest k,
Reading Q23: a row with no available primary action gets act = -1 for the primary, no read
heads and logp = 0 (parameter heads are still drawn).
With u drawn by the counter-based generator both sides implement:
    u(b, k) = ((splitmix64(seed + (step << 32) + 1024 b + k) >> 41) + 1/2) / 2^23
for row b and logit k (0..654, the concatenated head logits) -- 23 bits, so that every u is
exactly representable in binary32 as well (u <= 1 - 2^-24).
"""
import numpy as np

from .buffer import splitmix64, M64
from .loss import heads_forward, _masked_log_softmax
from .lstm import lstm_forward


def uniforms(seed: int, step: int, B: int, n_logits: int) -> np.ndarray:
    """u [B][n_logits] in (0, 1), the generator of reading Q22."""
    base = (seed + (step << 32)) & M64
    u = np.empty((B, n_logits))
    for b in range(B):
        for k in range(n_logits):
            z = splitmix64((base + 1024 * b + k) & M64)
            u[b, k] = ((z >> 41) + 0.5) / float(1 << 23)
    return u


def gumbel(u):
    """Gumbel(0, 1) noise from uniforms: g = -log(-log u)."""
    return -np.log(-np.log(np.asarray(u, np.float64)))


def sample(y, u, avail, head_table, head_sizes):
    """Masked factorised sampling from head outputs y [B][A] with uniforms u [B][n_logits]
    (reading Q22).  Returns act, head_on, logp, score."""
    y = np.asarray(y, np.float64)
    B = y.shape[0]
    n_logits = sum(head_sizes)
    g = gumbel(u)
    avail = np.asarray(avail).astype(bool)
    table = np.asarray(head_table).astype(bool)
    act = np.zeros((B, len(head_sizes)), np.int64)
    score = np.full((B, n_logits), -np.inf)
    off = np.concatenate([[0], np.cumsum(head_sizes)])
    lps = []
    for k, n in enumerate(head_sizes):
        lk = y[:, off[k]:off[k + 1]]
        allowed = avail if k == 0 else np.ones_like(lk, bool)   # action filters
        s = np.where(allowed, lk + g[:, off[k]:off[k + 1]], -np.inf)
        score[:, off[k]:off[k + 1]] = s
        act[:, k] = np.argmax(s, axis=1)          # first maximum on ties
        with np.errstate(divide="ignore", invalid="ignore"):   # rows with nothing allowed
            lps.append(_masked_log_softmax(lk, allowed))
    none = ~avail.any(axis=1)                     # reading Q23: no available primary
    act[none, 0] = -1
    head_on = np.where(none[:, None], False, table[np.maximum(act[:, 0], 0)])
    logp = np.zeros(B)
    for k in range(len(head_sizes)):
        on = head_on[:, k]
        sel = lps[k][np.arange(B), np.maximum(act[:, k], 0)]
        logp += np.where(on, sel, 0.0)            # ignored heads do not count
    return act, head_on.astype(np.uint8), logp, score


def infer_step(params, x, h, c, avail, head_table, seed, step, head_sizes):
    """params: canonical Wx, Wh, b, Wo, bo; x [B][D]; h, c [B][H]; avail [B][n_primary];
    head_table [n_primary][n_heads].  Returns dict h, c (new state), y [B][A] (logits |
    value), act [B][n_heads], head_on [B][n_heads], logp [B], value [B], score (the
    Gumbel-perturbed logits, -inf where not allowed) for validity checks."""
    x = np.asarray(x, np.float64)
    B = x.shape[0]
    # one LSTM step from the carried state
    st = lstm_forward(params["Wx"], params["Wh"], params["b"], x[None], h, c)
    h1, c1 = st["h"][0], st["c"][0]
    # heads
    y = heads_forward(h1, params["Wo"], params["bo"])
    u = uniforms(seed, step, B, sum(head_sizes))
    act, head_on, logp, score = sample(y, u, avail, head_table, head_sizes)
    return dict(h=h1, c=c1, y=y, act=act, head_on=head_on, logp=logp, value=y[:, -1],
                score=score)
