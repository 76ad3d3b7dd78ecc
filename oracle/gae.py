"""ORACLE (test infrastructure only) -- discount and Generalized Advantage Estimation.

P:1244 [§3.2] "The optimization algorithm uses Generalized Advantage Estimation (GAE)";
P:913 [Table hyperparams] GAE lambda = 0.95; P:1269 [§3.2] 256-step segments;
P:1525-1529 [§4.5, Eq. horizon] H = T / (1 - gamma).
"""
import numpy as np


def gamma_from_horizon(horizon_s: float, T_step: float = 4.0 / 30.0) -> float:
    """Eq. horizon: H = T/(1-gamma)  =>  gamma = 1 - T/H.
    T = 4 frames at 30 fps; the paper prints T = 0.133 s."""
    return 1.0 - T_step / horizon_s


def gae(r, V, done, gamma, lam):
    """GAE over rollout streams (DESIGN O2, reading Q10).

    r    [R][L]   rewards
    V    [R][L+1] value estimates; V[:, L] is the bootstrap value
    done [R][L]   1 if the episode ended after step t (zeroes bootstrap and carry)

    For t = L-1 ... 0:
        delta_t = r_t + gamma (1 - d_t) V_{t+1} - V_t
        A_t     = delta_t + gamma lam (1 - d_t) A_{t+1},   A_L = 0
        R_t     = A_t + V_t
    Returns (A, R) as float64 [R][L].
    """
    r = np.asarray(r, np.float64)
    V = np.asarray(V, np.float64)
    d = np.asarray(done, np.float64)
    gamma = float(gamma)
    lam = float(lam)
    R_, L = r.shape
    A = np.zeros((R_, L))
    a_next = np.zeros(R_)
    for t in reversed(range(L)):
        nd = 1.0 - d[:, t]
        delta = r[:, t] + gamma * nd * V[:, t + 1] - V[:, t]
        a = delta + gamma * lam * nd * a_next
        A[:, t] = a
        a_next = a
    return A, A + V[:, :L]


def segments_to_sequences(a, T):
    """DESIGN O3: sequence (r, k) is steps kT ... kT+T-1 of stream r; the minibatch
    is time-major [T][B] with sequence index b = r*(L/T) + k."""
    a = np.asarray(a)
    R_, L = a.shape
    assert L % T == 0
    return a.reshape(R_, L // T, T).reshape(R_ * (L // T), T).T.copy()
