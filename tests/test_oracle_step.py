"""Pins for the composed oracle step: end-to-end finite differences and DP averaging."""
import numpy as np

import oracle
from oracle.step import loss_and_grads
import synth


def _setup(seed, B=3, T=4, H=4, D=8, bo_scale=0.1):
    cfg = synth.Config(H=H, D=D, B=B, T=T)
    p = {k: v.astype(np.float64) for k, v in synth.make_params(cfg, seed, bo_scale).items()}
    p["Wo"] *= 30.0  # make the heads matter at this tiny H
    seq = synth.make_sequences(cfg, seed, pad_frac=0.3)
    rng = np.random.default_rng(seed)
    adv = rng.standard_normal((T, B))
    ret = rng.standard_normal((T, B))
    lp0 = loss_and_grads(p, seq, np.zeros((T, B)), adv, ret, cfg.head_sizes)[3]["logpi"]
    logp_old = lp0.reshape(T, B) + seq["logp_noise"]
    return cfg, p, seq, logp_old, adv, ret


def test_step_finite_differences():
    for seed in range(20):
        cfg, p, seq, logp_old, adv, ret = _setup(seed)
        rho = np.exp(loss_and_grads(p, seq, logp_old, adv, ret, cfg.head_sizes)[3]["logpi"]
                     - logp_old.reshape(-1))
        if np.all(np.minimum(np.abs(rho - 0.8), np.abs(rho - 1.2)) > 1e-3):
            break
    L0, g, _, _ = loss_and_grads(p, seq, logp_old, adv, ret, cfg.head_sizes)
    rng = np.random.default_rng(0)
    eps = 1e-6
    for name in ("Wx", "Wh", "b", "Wo", "bo"):
        P = p[name]
        for _ in range(12):
            idx = tuple(rng.integers(0, s) for s in P.shape)
            pp = dict(p)
            pm = dict(p)
            pp[name] = P.copy()
            pm[name] = P.copy()
            pp[name][idx] += eps
            pm[name][idx] -= eps
            fd = (loss_and_grads(pp, seq, logp_old, adv, ret, cfg.head_sizes)[0]
                  - loss_and_grads(pm, seq, logp_old, adv, ret, cfg.head_sizes)[0]) / (2 * eps)
            assert abs(fd - g[name][idx]) <= 1e-8 + 1e-6 * abs(fd), (name, idx, fd, g[name][idx])


def test_dp_average_of_equal_shards_equals_full_batch():
    """P:1251 average of per-GPU gradients == gradient of the concatenated batch when every
    shard uses its local denominator T*B/N (DESIGN Q9)."""
    cfg, p, seq, logp_old, adv, ret = _setup(3, B=8)
    _, g_full, _, _ = loss_and_grads(p, seq, logp_old, adv, ret, cfg.head_sizes)
    N = 4
    shards = []
    for n in range(N):
        sl = slice(n * 2, (n + 1) * 2)
        sub = {k: (v[:, sl] if v.ndim >= 2 and k not in ("h0", "c0") else v[sl]) for k, v in seq.items()}
        shards.append(loss_and_grads(p, sub, logp_old[:, sl], adv[:, sl], ret[:, sl],
                                     cfg.head_sizes)[1])
    avg = oracle.dp_average(shards)
    for k in g_full:
        np.testing.assert_allclose(avg[k], g_full[k], rtol=1e-12, atol=1e-15)


def test_dp_identical_shards():
    cfg, p, seq, logp_old, adv, ret = _setup(4)
    _, g, _, _ = loss_and_grads(p, seq, logp_old, adv, ret, cfg.head_sizes)
    avg = oracle.dp_average([g, g, g])
    for k in g:
        np.testing.assert_allclose(avg[k], g[k], rtol=1e-15, atol=0)


def test_full_step_runs_and_moves_params():
    cfg, p, seq, logp_old, adv, ret = _setup(5, B=4, T=4)
    ro = synth.make_rollouts(1, 16, 5)
    conf = dict(gamma=oracle.gamma_from_horizon(180.0), lam=0.95, clip_eps=0.2, c_v=1.0, c_e=0.01,
                lr=5e-5, beta1=0.9, beta2=0.999, adam_eps=1e-8, clip_sigma=5.0,
                head_sizes=cfg.head_sizes)
    state = {k: (np.zeros_like(v), np.zeros_like(v)) for k, v in p.items()}
    newp, newstate, rec = oracle.ppo_step(p, state, seq, ro, logp_old, conf, 1)
    assert rec["adv"].shape == (4, 4)
    for k in p:
        d = newp[k] - p[k]
        assert np.all(np.abs(d) <= 5e-5 * 1.0001)


def _gae_double_sum(r, V, d, gamma, lam):
    """A_t = sum_l (gamma lam)^l delta_{t+l}, stopping at the first done (Q10)."""
    L = r.shape[0]
    delta = [r[t] + (0.0 if d[t] else gamma * V[t + 1]) - V[t] for t in range(L)]
    A = np.zeros(L)
    for t in range(L):
        for l in range(L - t):
            A[t] += (gamma * lam) ** l * delta[t + l]
            if d[t + l]:
                break
    return A


def test_ppo_step_first_update_closed_form():
    """oracle.ppo_step end to end (GAE -> sequences -> loss gradient -> Adam), pinned by
    pieces that share nothing with it: GAE by its double sum, the sequence layout written
    out (sequence b = k-th T-window of the stream, time-major), the gradient of the loss by
    central finite differences, and Adam's first step from a zero state in closed form
    (DESIGN Q3/Q4): v = (1-b2) g^2, g_c = clip(g, +-5 sqrt(v)) = 5 sqrt(1-b2) g
    (5 sqrt(1-b2) < 1), m = (1-b1) g_c, alpha_1 = lr sqrt(1-b2) / (1-b1), so
        dtheta = -lr 5 (1-b2) g / (sqrt(1-b2) |g| + eps).
    A transposed layout, a gradient of the wrong sign or shard, or Adam state mixed between
    tensors fails it."""
    conf = dict(gamma=oracle.gamma_from_horizon(180.0), lam=0.95, clip_eps=0.2, c_v=1.0,
                c_e=0.01, lr=5e-5, beta1=0.9, beta2=0.999, adam_eps=1e-8, clip_sigma=5.0)
    T = 4
    for seed in range(5, 40):
        cfg, p, seq, logp_old, _, _ = _setup(seed, B=4, T=T)
        ro = synth.make_rollouts(1, 16, seed, p_done=0.15)
        r, V, d = (np.asarray(ro[k], np.float64)[0] for k in ("r", "V", "done"))
        A = _gae_double_sum(r, V, d, conf["gamma"], conf["lam"])
        adv = np.zeros((T, 4))
        ret = np.zeros((T, 4))
        for k in range(4):
            for t in range(T):
                adv[t, k] = A[k * T + t]
                ret[t, k] = A[k * T + t] + V[k * T + t]
        lp = loss_and_grads(p, seq, logp_old, adv, ret, cfg.head_sizes)[3]["logpi"]
        rho = np.exp(lp - logp_old.reshape(-1))
        if np.all(np.minimum(np.abs(rho - 0.8), np.abs(rho - 1.2)) > 1e-3) and d.any():
            break
    conf["head_sizes"] = cfg.head_sizes
    state = {k: (np.zeros_like(v), np.zeros_like(v)) for k, v in p.items()}
    newp, _, rec = oracle.ppo_step(p, state, seq, ro, logp_old, conf, 1)
    np.testing.assert_allclose(rec["adv"], adv, rtol=0, atol=1e-12)
    np.testing.assert_allclose(rec["ret"], ret, rtol=0, atol=1e-12)

    def loss(pp):
        return loss_and_grads(pp, seq, logp_old, adv, ret, cfg.head_sizes, 0.2, 1.0, 0.01)[0]

    rng = np.random.default_rng(1)
    b2, h = conf["beta2"], 1e-6
    checked = 0
    for name in ("Wx", "Wh", "b", "Wo", "bo"):
        P = p[name]
        for _ in range(10):
            idx = tuple(rng.integers(0, s) for s in P.shape)
            pp, pm = dict(p), dict(p)
            pp[name], pm[name] = P.copy(), P.copy()
            pp[name][idx] += h
            pm[name][idx] -= h
            g = (loss(pp) - loss(pm)) / (2 * h)
            if abs(g) < 1e-6:      # finite-difference noise would decide the sign
                continue
            want = -conf["lr"] * 5.0 * (1 - b2) * g / (np.sqrt(1 - b2) * abs(g) + 1e-8)
            got = newp[name][idx] - P[idx]
            assert abs(got - want) <= 1e-4 * abs(want), (name, idx, got, want, g)
            checked += 1
    assert checked >= 25
