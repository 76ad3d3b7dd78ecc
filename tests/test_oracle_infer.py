"""Pins for the NEXT-3 inference oracle (oracle/infer.py, reading Q22).

What pins it to something other than itself:
  * the carried state: two inference steps == the (pinned) LSTM oracle over a 2-step sequence;
  * Gumbel-max: empirical action frequencies over many counter draws == softmax probabilities
    (chi-square), which a sign or direction error in g = -log(-log u) fails;
  * the generator: u strictly inside (0, 1), 23-bit grid exact in binary32, moments of U(0, 1);
  * masks: an unavailable primary is never drawn, a lone available one always (log p = 0);
  * bookkeeping: head_on = table[primary]; logp == the (pinned) loss oracle's log pi of the
    sampled actions; inactive heads add nothing.
"""
import numpy as np
import pytest

import synth
from oracle import infer as oi
from oracle.loss import ppo_loss
from oracle.lstm import lstm_forward

CFG = synth.Config(H=32, D=48, B=6, T=2)


def _params(seed=0):
    p = synth.make_params(CFG, seed, bo_scale=0.3)
    p["Wo"] = p["Wo"] * 100.0      # logits O(1): the sampler sees real preferences
    return p


def _state(seed=1):
    s = synth.make_sequences(CFG, seed)
    return s


def test_state_carry_equals_two_step_lstm():
    p, s = _params(), _state()
    tab = synth.heads_on_table(CFG.head_sizes)
    st = dict(h=s["h0"], c=s["c0"])
    for t in range(2):
        st = oi.infer_step(p, s["x"][t], st["h"], st["c"], s["avail"][t], tab, 7, t,
                           CFG.head_sizes)
    ref = lstm_forward(p["Wx"], p["Wh"], p["b"], s["x"], s["h0"], s["c0"])
    assert np.allclose(st["h"], ref["h"][1], rtol=0, atol=1e-13)
    assert np.allclose(st["c"], ref["c"][1], rtol=0, atol=1e-13)
    assert np.allclose(st["value"], st["y"][:, -1])


def test_uniform_generator():
    u = oi.uniforms(123, 5, 40, 655)
    assert u.min() > 0.0 and u.max() < 1.0
    # 23-bit grid: (j + 1/2) / 2^23, every value exact in binary32
    j = u * (1 << 23) - 0.5
    assert np.array_equal(j, np.round(j))
    assert np.array_equal(u.astype(np.float32).astype(np.float64), u)
    assert abs(u.mean() - 0.5) < 0.01 and abs(u.var() - 1.0 / 12) < 0.005
    # distinct rows / steps give distinct draws; same counter gives the same draw
    assert not np.array_equal(u[0], u[1])
    assert np.array_equal(u, oi.uniforms(123, 5, 40, 655))
    assert not np.array_equal(u, oi.uniforms(123, 6, 40, 655))


def test_gumbel_max_samples_the_softmax():
    """A 4-way head with fixed logits: frequencies over 40,000 draws match softmax."""
    logits = np.array([0.3, -1.2, 1.5, 0.0])
    p = np.exp(logits - logits.max())
    p /= p.sum()
    hs = (4,)
    n = 40000
    u = oi.uniforms(99, 0, n, 4)   # rows are independent draws
    act, _, _, _ = oi.sample(np.tile(np.append(logits, 0.0), (n, 1)), u,
                             np.ones((n, 4), np.uint8), np.ones((4, 1), np.uint8), hs)
    counts = np.bincount(act[:, 0], minlength=4)
    chi2 = ((counts - n * p) ** 2 / (n * p)).sum()
    assert chi2 < 16.27, (counts, n * p, chi2)   # 3 dof, p = 0.001


def test_primary_mask_and_lone_action():
    hs = CFG.head_sizes
    B = 200
    rng = np.random.default_rng(0)
    y = rng.standard_normal((B, sum(hs) + 1))
    avail = (rng.random((B, hs[0])) < 0.3).astype(np.uint8)
    avail[:, 0] = 1
    avail[:50] = 0
    avail[np.arange(50), np.arange(50) % hs[0]] = 1      # one available action only
    tab = synth.heads_on_table(hs)
    u = oi.uniforms(3, 1, B, sum(hs))
    act, head_on, logp, score = oi.sample(y, u, avail, tab, hs)
    assert np.all(avail[np.arange(B), act[:, 0]] == 1)
    assert np.array_equal(act[:50, 0], np.arange(50) % hs[0])
    assert np.array_equal(head_on, tab[act[:, 0]])
    # lone primary: log p(primary) = 0, so logp = the read parameter heads only
    only_primary = np.zeros_like(tab)
    only_primary[:, 0] = 1
    _, _, lp1, _ = oi.sample(y, u, avail, only_primary, hs)
    assert np.allclose(lp1[:50], 0.0, atol=1e-12)
    assert np.all(lp1[50:] < 0)
    # argmax of the scores, scores -inf only where not allowed
    off = np.concatenate([[0], np.cumsum(hs)])
    for k in range(len(hs)):
        sk = score[:, off[k]:off[k + 1]]
        assert np.array_equal(act[:, k], sk.argmax(1))
    assert np.array_equal(np.isinf(score[:, :hs[0]]), avail == 0)


def test_no_available_primary():
    hs = CFG.head_sizes
    rng = np.random.default_rng(1)
    y = rng.standard_normal((3, sum(hs) + 1))
    avail = np.ones((3, hs[0]), np.uint8)
    avail[1] = 0
    act, head_on, logp, _ = oi.sample(y, oi.uniforms(0, 0, 3, sum(hs)), avail,
                                      synth.heads_on_table(hs), hs)
    assert act[1, 0] == -1 and not head_on[1].any() and logp[1] == 0.0
    assert act[0, 0] >= 0 and head_on[0, 0] == 1 and logp[0] < 0
    assert np.all(act[1, 1:] >= 0)


def test_logp_equals_loss_oracle_log_pi():
    """The behaviour log-prob the sampler returns is the loss oracle's log pi of the same
    actions and read heads (it is what the PPO ratio divides by)."""
    p, s = _params(2), _state(3)
    tab = synth.heads_on_table(CFG.head_sizes)
    r = oi.infer_step(p, s["x"][0], s["h0"], s["c0"], s["avail"][0], tab, 11, 0, CFG.head_sizes)
    B = CFG.B
    _, _, _, logpi = ppo_loss(r["y"], r["act"], r["head_on"], s["avail"][0], np.zeros(B),
                              np.zeros(B), np.zeros(B), np.ones(B), CFG.head_sizes)
    assert np.allclose(r["logp"], logpi, rtol=0, atol=1e-12)


@pytest.mark.parametrize("B", [1, 7])
def test_deterministic_in_counter(B):
    p = _params(4)
    cfg = synth.Config(H=CFG.H, D=CFG.D, B=B, T=1)
    s = synth.make_sequences(cfg, 5)
    tab = synth.heads_on_table(CFG.head_sizes)
    a = oi.infer_step(p, s["x"][0], s["h0"], s["c0"], s["avail"][0], tab, 1, 2, CFG.head_sizes)
    b = oi.infer_step(p, s["x"][0], s["h0"], s["c0"], s["avail"][0], tab, 1, 2, CFG.head_sizes)
    assert np.array_equal(a["act"], b["act"]) and np.array_equal(a["logp"], b["logp"])
