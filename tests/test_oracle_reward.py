"""Pins for oracle.reward (NEXT-2): the closed forms the paper's reward pieces reduce to."""
import numpy as np

from oracle import reward


def _raw(seed, G=3, L=50):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((G, 10, L)), (rng.uniform(0, 1, (G, 10, L)) < 0.01) * 5.0


def test_identity_when_pieces_off():
    sh, win = _raw(0)
    r = reward.shape_rewards(sh, win, np.zeros(3), tau=0.0, decay_base=1.0, zero_sum=False)
    np.testing.assert_allclose(r, sh + win, rtol=0, atol=0)


def test_team_spirit_one_shares_equally():
    # "If team spirit is 1, then every reward is split equally among all five heroes"
    sh, win = _raw(1)
    r = reward.shape_rewards(sh, win, np.zeros(3), tau=1.0, zero_sum=False)
    for team in (slice(0, 5), slice(5, 10)):
        assert np.allclose(r[:, team], r[:, team][:, :1], atol=1e-15)


def test_zero_sum_total_is_zero():
    # everything that benefits one team hurts the other: the 10 rewards sum to 0
    sh, win = _raw(2)
    for tau in (0.0, 0.3, 0.8, 1.0):
        r = reward.shape_rewards(sh, win, np.array([0, 100, 7000]), tau=tau)
        assert np.abs(r.sum(axis=1)).max() < 1e-12


def test_time_decay_at_ten_minutes_and_win_exempt():
    # Eq. P:1066: rho <- rho * 0.6^(T/10 min); 10 min = 4500 steps of 4/30 s; win exempt
    G, L = 1, 3
    sh = np.ones((G, 10, L))
    win = np.zeros((G, 10, L))
    win[0, 0, 0] = 5.0
    r = reward.shape_rewards(sh, win, np.array([4500]), tau=0.0, zero_sum=False)
    assert abs(r[0, 1, 0] - 0.6) < 1e-12
    assert abs(r[0, 0, 0] - (0.6 + 5.0)) < 1e-12
    assert abs(r[0, 1, 1] - 0.6 ** (4501 / 4500)) < 1e-12


def test_running_std_merge_equals_concatenation():
    rng = np.random.default_rng(3)
    xs = [rng.standard_normal(n) * 2 + 0.5 for n in (10, 1000, 37)]
    stats = (0, 0.0, 0.0)
    sigmas = []
    for x in xs:
        s, stats = reward.running_std_update(stats, x)
        sigmas.append(s)
    assert sigmas[0] == 1.0
    assert abs(sigmas[1] - np.std(xs[0])) < 1e-12
    assert abs(sigmas[2] - np.std(np.concatenate(xs[:2]))) < 1e-12
    allx = np.concatenate(xs)
    assert stats[0] == allx.size and abs(stats[1] - allx.mean()) < 1e-12
    assert abs(stats[2] / stats[0] - allx.var()) < 1e-12
