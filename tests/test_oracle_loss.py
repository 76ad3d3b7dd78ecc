"""Pins for oracle.loss: PPO clip invariants, entropy closed forms, masking, finite differences."""
import math

import numpy as np
import pytest

import oracle
import synth

HS = synth.HEAD_SIZES
A = synth.A_OUT


def _batch(seed, rows=24, scale=1.0, pad=False):
    cfg = synth.Config(H=8, D=8, B=rows, T=1)
    s = synth.make_sequences(cfg, seed, pad_frac=0.5 if pad else 0.0)
    Y = synth.make_logits(rows, A, seed, scale)
    rng = np.random.default_rng(seed + 100)
    adv = rng.standard_normal(rows)
    ret = rng.standard_normal(rows)
    return Y, s["act"][0], s["head_on"][0], s["avail"][0], s["valid"][0], adv, ret


def _logpi(Y, act, on, av):
    return oracle.ppo_loss(Y, act, on, av, np.zeros(len(Y)), np.zeros(len(Y)), np.zeros(len(Y)),
                           None, HS, c_v=0, c_e=0)[3]


@pytest.mark.parametrize("seed", range(4))
def test_rho_one_gives_minus_mean_advantage(seed):
    Y, act, on, av, _, adv, ret = _batch(seed)
    lp = _logpi(Y, act, on, av)
    L, dY, st, _ = oracle.ppo_loss(Y, act, on, av, lp, adv, ret, None, HS, c_v=0, c_e=0)
    assert abs(L - (-adv.mean())) < 1e-13
    assert abs(st["clipfrac"]) == 0 and abs(st["approx_kl"]) < 1e-13


@pytest.mark.parametrize("rho,sign,clipped_val,zero_grad", [
    (1.5, +1, 1.2, True),    # rho=1.5, A>0 -> 1.2 A, clipped side
    (0.5, -1, 0.8, True),    # A<0, rho<1-eps -> clipped at 0.8, zero gradient
    (0.5, +1, 0.5, False),   # A>0, rho<1-eps -> unclipped (min picks rho A)
    (1.5, -1, 1.5, False),   # A<0, rho>1+eps -> unclipped
])
def test_clip_invariants(rho, sign, clipped_val, zero_grad):
    Y, act, on, av, _, adv, ret = _batch(5)
    adv = sign * np.abs(adv) + sign * 0.1
    lp = _logpi(Y, act, on, av)
    L, dY, st, _ = oracle.ppo_loss(Y, act, on, av, lp - math.log(rho), adv, ret, None, HS,
                                   c_v=0, c_e=0)
    assert abs(L - np.mean(-clipped_val * adv)) < 1e-12
    logits = dY[:, :-1]
    if zero_grad:
        assert np.all(logits == 0.0)
        assert st["clipfrac"] == 1.0
    else:
        assert np.abs(logits).max() > 1e-3
        assert st["clipfrac"] == 0.0


def test_uniform_policy_entropy_is_log_m():
    Y, act, on, av, _, adv, ret = _batch(2)
    Y = np.zeros_like(Y)
    _, _, st, _ = oracle.ppo_loss(Y, act, on, av, np.zeros(len(Y)), adv, ret, None, HS,
                                  c_v=0, c_e=1.0)
    expect = 0.0
    for r in range(len(Y)):
        expect += math.log(av[r].sum()) + sum(on[r, k] * math.log(HS[k]) for k in range(1, len(HS)))
    assert abs(st["ent"] - expect / len(Y)) < 1e-12


def test_masking_exact_zeros():
    """Unavailable primaries get probability exactly 0 and gradient exactly 0;
    heads ignored by the chosen primary get gradient exactly 0."""
    Y, act, on, av, _, adv, ret = _batch(3)
    lp = _logpi(Y, act, on, av)
    _, dY, _, _ = oracle.ppo_loss(Y, act, on, av, lp + 0.05, adv, ret, None, HS)
    offs = np.concatenate([[0], np.cumsum(HS)])
    assert np.all(dY[:, :HS[0]][av == 0] == 0.0)
    for k in range(1, len(HS)):
        rows_off = on[:, k] == 0
        assert np.all(dY[rows_off, offs[k]:offs[k + 1]] == 0.0)
        assert np.any(dY[~rows_off, offs[k]:offs[k + 1]] != 0.0) or not np.any(~rows_off)


def test_invalid_rows_contribute_nothing():
    Y, act, on, av, valid, adv, ret = _batch(4, pad=True)
    assert valid.min() == 0 and valid.max() == 1
    lp = _logpi(Y, act, on, av) + 0.03
    L, dY, st, _ = oracle.ppo_loss(Y, act, on, av, lp, adv, ret, valid, HS)
    assert np.all(dY[valid == 0] == 0.0)
    keep = valid == 1
    L2, _, _, _ = oracle.ppo_loss(Y[keep], act[keep], on[keep], av[keep], lp[keep], adv[keep],
                                  ret[keep], None, HS, denom=float(len(Y)))
    assert abs(L - L2) < 1e-13
    assert st["n_valid"] == keep.sum()


@pytest.mark.parametrize("seed", range(3))
def test_finite_differences(seed):
    Y, act, on, av, valid, adv, ret = _batch(seed, rows=6, scale=0.7)
    rng = np.random.default_rng(seed)
    lp = _logpi(Y, act, on, av) + 0.1 * rng.standard_normal(len(Y))
    rho = np.exp(_logpi(Y, act, on, av) - lp)
    assert np.all(np.minimum(np.abs(rho - 0.8), np.abs(rho - 1.2)) > 1e-3)

    def L(Y_):
        return oracle.ppo_loss(Y_, act, on, av, lp, adv, ret, valid, HS, c_e=0.3)[0]

    _, dY, _, _ = oracle.ppo_loss(Y, act, on, av, lp, adv, ret, valid, HS, c_e=0.3)
    eps = 1e-6
    idxs = [(r, c) for r in range(len(Y)) for c in range(0, A, 7)] + [(r, A - 1) for r in range(len(Y))]
    for r, c in idxs:
        Yp, Ym = Y.astype(np.float64).copy(), Y.astype(np.float64).copy()
        Yp[r, c] += eps
        Ym[r, c] -= eps
        fd = (L(Yp) - L(Ym)) / (2 * eps)
        assert abs(fd - dY[r, c]) <= 1e-7 + 1e-6 * abs(fd), (r, c, fd, dY[r, c])
