"""ORACLE (test infrastructure only) -- NEXT-4: the auxiliary prediction heads.

App. Evaluating agents' understanding: "small networks of fully-connected
layers that transform LSTM output into predictions" of
  * win probability -- binary label, 0 or 1 at the end of the game;
  * net worth rank -- the hero's rank (1-5) within its team at the end of the game;
  * team objectives / enemy buildings -- whether the hero will help destroy a given enemy
    building in the near future, with "an additional discount factor with horizon
    of 2 minutes".
"win probability passes gradients to the main LSTM and rest of the agent with a very small
weight; the other auxiliary predictions use ... stop_gradient".
Labels (Eq.): for a segment t1..t2, y = the ground truth on the last segment of
the game, else the model's prediction y_hat(t2) at the end of the segment.

Readings (Q24-Q27):
  Q24 each aux head is one linear projection of the LSTM output (like the value head),
      appended after the value: y = [policy logits | V | win (n_win) | rank (n_rank) |
      buildings (n_bld)]; win and buildings are logistic, rank is a softmax over n_rank.
  Q25 losses: binary cross-entropy (win, each building), cross-entropy against the (possibly
      soft, bootstrapped) rank distribution; weights c_win, c_rank, c_bld; same valid mask
      and T*B denominator as the PPO loss (Q9); L = L_ppo + L_aux.
  Q26 routing: every aux head's own weights get the full gradient of its loss; the LSTM
      receives win_trunk x the win head's gradient and nothing from the other aux heads.
  Q27 labels per 256-step segment (steps 0..L-1, bootstrap y_hat after step L-1):
      win  y_t = outcome if last else y_hat_win;   rank y_t = onehot(final rank) if last
      else y_hat_rank;  building j: y_t = 1 if the event happens at step t, else
      gamma2 * y_{t+1}, with y_L = 0 if last else y_hat_bld_j and gamma2 = 1 - T_step/120 s
      (the value discount's horizon formula, with a 2-minute horizon).
"""
import numpy as np


def aux_labels(last, outcome, rank, events, boot, gamma2, n_win, n_rank, n_bld):
    """last [R] bool, outcome [R] (0/1), rank [R] int in [0, n_rank), events [R][L][n_bld]
    (0/1), boot [R][n_win + n_rank + n_bld] (the model's predictions after the segment's last
    step).  Returns labels [R][L][n_aux] (Q27)."""
    events = np.asarray(events)
    R, L = events.shape[0], events.shape[1]
    boot = np.asarray(boot, np.float64)
    n_aux = n_win + n_rank + n_bld
    y = np.zeros((R, L, n_aux))
    for r in range(R):
        c = 0
        if n_win:
            y[r, :, 0] = float(outcome[r]) if last[r] else boot[r, 0]
            c = 1
        if n_rank:
            if last[r]:
                y[r, :, c + int(rank[r])] = 1.0
            else:
                y[r, :, c:c + n_rank] = boot[r, c:c + n_rank]
            c += n_rank
        for j in range(n_bld):
            nxt = 0.0 if last[r] else boot[r, c + j]
            for t in reversed(range(L)):
                nxt = 1.0 if events[r, t, j] else gamma2 * nxt
                y[r, t, c + j] = nxt
    return y


def _softplus(z):
    return np.maximum(z, 0.0) + np.log1p(np.exp(-np.abs(z)))


def _sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def aux_loss(Yaux, labels, valid, n_win, n_rank, n_bld, c_win=1.0, c_rank=1.0, c_bld=1.0,
             denom=None):
    """Yaux [N][n_aux] aux head outputs, labels [N][n_aux], valid [N].  Returns
    (L_aux, dYaux [N][n_aux] -- the full gradient of L_aux, comps dict) (Q25)."""
    Y = np.asarray(Yaux, np.float64)
    lab = np.asarray(labels, np.float64)
    N = Y.shape[0]
    w = np.ones(N) if valid is None else np.asarray(valid, np.float64)
    d = float(N) if denom is None else float(denom)
    dY = np.zeros_like(Y)
    comps = dict(win=0.0, rank=0.0, bld=0.0)
    c = 0
    if n_win:
        z, y = Y[:, 0], lab[:, 0]
        comps["win"] = float(np.sum(w * (_softplus(z) - y * z)) / d)   # BCE(sigma(z), y)
        dY[:, 0] = c_win * w * (_sigmoid(z) - y) / d
        c = 1
    if n_rank:
        z, y = Y[:, c:c + n_rank], lab[:, c:c + n_rank]
        m = z.max(axis=1, keepdims=True)
        lse = m + np.log(np.exp(z - m).sum(axis=1, keepdims=True))
        logp = z - lse
        comps["rank"] = float(np.sum(w * -(y * logp).sum(axis=1)) / d)
        p = np.exp(logp)
        dY[:, c:c + n_rank] = c_rank * (w / d)[:, None] * (p * y.sum(axis=1, keepdims=True) - y)
        c += n_rank
    if n_bld:
        z, y = Y[:, c:c + n_bld], lab[:, c:c + n_bld]
        comps["bld"] = float(np.sum(w[:, None] * (_softplus(z) - y * z)) / d)
        dY[:, c:c + n_bld] = c_bld * (w / d)[:, None] * (_sigmoid(z) - y)
    L = c_win * comps["win"] + c_rank * comps["rank"] + c_bld * comps["bld"]
    return L, dY, comps


def trunk_gradient(dYaux, n_win, win_trunk):
    """Q26: the part of the aux gradient that reaches the LSTM output: win_trunk x the win
    column, zero for the stop_gradient heads."""
    g = np.zeros_like(np.asarray(dYaux, np.float64))
    if n_win:
        g[:, 0] = win_trunk * np.asarray(dYaux)[:, 0]
    return g
