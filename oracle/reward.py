"""ORACLE (test infrastructure only) -- NEXT-2: the reward pipeline in front of GAE.

App. Reward Weights: every hero's shaped reward is
  * game-time weighted: rho_i <- rho_i * 0.6^(T / 10 min), for all rewards other than win/loss
    (Eq.);
  * team-spirit mixed: r_i = (1 - tau) rho_i + tau * mean_team(rho)  (Eq.);
  * zero-sum: the average of the enemies' rewards is subtracted from each hero.
P:926 [Table hyperparams note c]: rewards are normalised by a running estimate of their
standard deviation (and the value loss weight applies post-normalisation).
Readings (DESIGN Q20, Q21): heroes 0-4 are one team, 5-9 the other; the three linear pieces
are applied in the order written above (they commute except that win/loss escapes the time
weighting); the running std is the population std of all final per-step rewards of the
PREVIOUS calls (Chan et al. parallel merge; sigma = 1 before any data), and this call's
rewards are divided by it, then folded into the running statistics.
"""
import numpy as np

T_STEP = 4.0 / 30.0   # seconds per policy step
TEN_MIN = 600.0


def shape_rewards(shaped, win, step0, tau, decay_base=0.6, zero_sum=True):
    """shaped, win: [G][10][L] raw per-hero rewards; step0: [G] game step of the first entry.
    Returns final per-hero rewards r [G][10][L] before normalisation."""
    shaped = np.asarray(shaped, np.float64)
    win = np.asarray(win, np.float64)
    G, NH, L = shaped.shape
    assert NH == 10
    t = (np.asarray(step0, np.float64)[:, None] + np.arange(L)[None, :]) * T_STEP  # [G][L] s
    rho = shaped * decay_base ** (t / TEN_MIN)[:, None, :] + win
    r = np.empty_like(rho)
    for team, enemy in ((slice(0, 5), slice(5, 10)), (slice(5, 10), slice(0, 5))):
        mean_team = rho[:, team].mean(axis=1, keepdims=True)
        r[:, team] = (1.0 - tau) * rho[:, team] + tau * mean_team
        if zero_sum:
            r[:, team] -= rho[:, enemy].mean(axis=1, keepdims=True)
    return r


def running_std_update(stats, x):
    """stats = (count, mean, M2) of all previous data; returns (sigma_prev, new stats).
    Chan, Golub & LeVeque pairwise merge of the batch x into the running moments."""
    count, mean, m2 = stats
    sigma = np.sqrt(m2 / count) if count > 0 else 1.0
    x = np.asarray(x, np.float64).reshape(-1)
    nb = x.size
    mb = x.mean()
    m2b = ((x - mb) ** 2).sum()
    n = count + nb
    delta = mb - mean
    new_mean = mean + delta * nb / n
    new_m2 = m2 + m2b + delta * delta * count * nb / n
    return sigma, (n, new_mean, new_m2)
