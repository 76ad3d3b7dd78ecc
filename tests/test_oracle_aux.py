"""Pins for the NEXT-4 aux-head oracle (oracle/aux.py, Q24-Q27).

  * labels: the paper's piecewise equation on hand-made segments; the 2-minute
    discount in closed form (gamma2^(e - t) before an event, bootstrap gamma2^(L - t) y_hat);
    gamma2 from the horizon formula and (1 - 1/n)^n ~ 1/e over its horizon;
  * losses: BCE at z = 0 is ln 2, uniform rank logits give ln n_rank, a one-hot rank label
    gives -log softmax; finite differences of L_aux in the head outputs;
  * routing: finite differences of the composed step -- the LSTM weights see
    L_ppo + win_trunk * c_win * L_win only, the aux rows of W_o see the whole L.
"""
import math

import numpy as np
import pytest

import synth
from oracle import aux as oa
from oracle.gae import gamma_from_horizon
from oracle.step import loss_and_grads

G2 = gamma_from_horizon(120.0)


def test_gamma2_horizon():
    assert abs(G2 - (1.0 - (4.0 / 30.0) / 120.0)) < 1e-15
    n = round(120.0 / (4.0 / 30.0))
    assert abs(G2 ** n - math.exp(-1.0)) < 1e-3


def test_labels_piecewise_and_discount():
    L, n_rank = 8, 3
    last = np.array([1, 1, 0, 0], bool)
    outcome = np.array([1.0, 0.0, 1.0, 0.0])
    rank = np.array([2, 0, 1, 1])
    events = np.zeros((4, L, 2), np.uint8)
    events[0, 5, 0] = 1              # last segment, event at step 5
    events[2, 3, 1] = 1              # not last, event at step 3
    events[2, 6, 1] = 1              # ... and again at 6
    boot = np.array([[0.3, 0.2, 0.3, 0.5, 0.7, 0.9],
                     [0.6, 0.1, 0.1, 0.8, 0.7, 0.9],
                     [0.25, 0.5, 0.25, 0.25, 0.4, 0.05],
                     [0.75, 0.0, 1.0, 0.0, 0.2, 0.1]])
    y = oa.aux_labels(last, outcome, rank, events, boot, G2, 1, n_rank, 2)
    assert y.shape == (4, L, 6)
    # win: ground truth on the game's last segment, else y_hat(t2), for every step
    assert np.all(y[0, :, 0] == 1.0) and np.all(y[1, :, 0] == 0.0)
    assert np.all(y[2, :, 0] == 0.25) and np.all(y[3, :, 0] == 0.75)
    # rank: one-hot of the final rank, else the predicted distribution
    assert np.array_equal(y[0, :, 1:4], np.tile([0, 0, 1.0], (L, 1)))
    assert np.array_equal(y[2, :, 1:4], np.tile(boot[2, 1:4], (L, 1)))
    t = np.arange(L)
    # building 0, last segment, event at 5: gamma2^(5-t) up to 5, then 0 (the game ended)
    np.testing.assert_allclose(y[0, :, 4], np.where(t <= 5, G2 ** (5 - t), 0.0), rtol=1e-15)
    # building 1 of segment 0 (no events, last): 0
    assert np.all(y[0, :, 5] == 0.0)
    # segment 2 building 1: nearest next event, bootstrap gamma2^(L-t) y_hat after the last
    exp = np.where(t <= 3, G2 ** (3 - t), np.where(t <= 6, G2 ** (6 - t), G2 ** (L - t) * 0.05))
    np.testing.assert_allclose(y[2, :, 5], exp, rtol=1e-15)
    # segment 3 (no events, not last): pure bootstrap
    np.testing.assert_allclose(y[3, :, 4], G2 ** (L - t) * 0.2, rtol=1e-15)


def test_loss_closed_forms():
    N = 5
    Y = np.zeros((N, 1 + 4 + 2))
    lab = np.zeros_like(Y)
    lab[:, 0] = 0.3
    lab[np.arange(N), 1 + np.arange(N) % 4] = 1.0
    lab[:, 5:] = 0.7
    L, dY, comps = oa.aux_loss(Y, lab, None, 1, 4, 2)
    assert abs(comps["win"] - math.log(2.0)) < 1e-15          # BCE(sigma(0), y) = ln 2
    assert abs(comps["rank"] - math.log(4.0)) < 1e-15         # uniform over 4 ranks
    assert abs(comps["bld"] - 2 * math.log(2.0)) < 1e-15
    assert abs(L - 3 * math.log(2.0) - math.log(4.0)) < 1e-14
    # one-hot rank label: -log softmax of the labelled class
    rng = np.random.default_rng(1)
    Y = rng.standard_normal((N, 7))
    L, dY, comps = oa.aux_loss(Y, lab, None, 1, 4, 2, c_win=0.0, c_rank=1.0, c_bld=0.0)
    z = Y[:, 1:5]
    ref = np.mean(-(z[np.arange(N), np.arange(N) % 4] - np.log(np.exp(z).sum(1))))
    assert abs(comps["rank"] - ref) < 1e-14 and abs(L - ref) < 1e-14


@pytest.mark.parametrize("seed", [0, 1])
def test_loss_finite_differences(seed):
    rng = np.random.default_rng(seed)
    N, sizes = 6, (1, 5, 3)
    Y = rng.standard_normal((N, sum(sizes)))
    lab = rng.uniform(0, 1, size=Y.shape)
    lab[:, 1:6] /= lab[:, 1:6].sum(1, keepdims=True)
    valid = (rng.random(N) < 0.7).astype(float)
    args = (valid, *sizes, 0.7, 1.3, 0.4, 9.0)
    L, dY, _ = oa.aux_loss(Y, lab, *args)
    eps = 1e-6
    for i in range(N):
        for j in range(Y.shape[1]):
            Yp, Ym = Y.copy(), Y.copy()
            Yp[i, j] += eps
            Ym[i, j] -= eps
            fd = (oa.aux_loss(Yp, lab, *args)[0] - oa.aux_loss(Ym, lab, *args)[0]) / (2 * eps)
            assert abs(fd - dY[i, j]) < 1e-8, (i, j, fd, dY[i, j])


def test_routing_finite_differences():
    """Trunk weights: gradient of L_ppo + win_trunk * c_win * L_win; aux rows of W_o: the
    gradient of the whole loss; stop_gradient heads reach the LSTM with nothing."""
    aux_sizes = (1, 3, 2)
    cfg = synth.Config(H=4, D=6, B=3, T=3, aux=aux_sizes)
    p = {k: v.astype(np.float64) for k, v in synth.make_params(cfg, 3, 0.1).items()}
    p["Wo"] *= 30.0
    seq = synth.make_sequences(cfg, 4, pad_frac=0.3)
    seq["avail"] = np.ones_like(seq["avail"])
    rng = np.random.default_rng(5)
    T, B = cfg.T, cfg.B
    adv, ret = rng.standard_normal((T, B)), rng.standard_normal((T, B))
    logp_old = rng.standard_normal((T, B)) - 1.0
    lab = rng.uniform(0, 1, size=(T, B, 6))
    lab[..., 1:4] /= lab[..., 1:4].sum(-1, keepdims=True)
    aux = dict(labels=lab, n_win=1, n_rank=3, n_bld=2, c_win=0.8, c_rank=1.1, c_bld=0.6,
               win_trunk=0.05)

    def run(pp):
        return loss_and_grads(pp, seq, logp_old, adv, ret, cfg.head_sizes, aux=aux)

    L0, g, st, _ = run(p)
    assert abs(st["loss"] - st["loss_ppo"] - st["aux"]) < 1e-14

    def surrogate(pp):   # what the LSTM is trained on (Q26)
        s = run(pp)[2]
        return s["loss_ppo"] + aux["win_trunk"] * aux["c_win"] * s["aux_win"]

    eps = 1e-6
    A0 = sum(cfg.head_sizes) + 1
    for name, f, rows in (("Wx", surrogate, None), ("Wh", surrogate, None), ("b", surrogate, None),
                          ("Wo", lambda pp: run(pp)[0], range(A0, cfg.A)),
                          ("bo", lambda pp: run(pp)[0], range(A0, cfg.A))):
        P = p[name]
        idxs = ([(r, c) for r in rows for c in range(P.shape[1])] if name == "Wo" and rows
                else [(r,) for r in rows] if rows else
                [tuple(rng.integers(0, s) for s in P.shape) for _ in range(10)])
        for idx in idxs:
            pp, pm = dict(p), dict(p)
            pp[name], pm[name] = P.copy(), P.copy()
            pp[name][idx] += eps
            pm[name][idx] -= eps
            fd = (f(pp) - f(pm)) / (2 * eps)
            assert abs(fd - g[name][idx]) <= 1e-8 + 1e-6 * abs(fd), (name, idx, fd, g[name][idx])
