"""Pins for oracle.gae against what the paper and the mathematics fix (CPU only)."""
import json
import os

import numpy as np
import pytest

import oracle
import synth


def test_spec_worked_example(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "gae_spec_example.json")))
    A, R = oracle.gae(np.array([g["r"]]), np.array([g["V"]]), np.array([g["done"]]),
                      g["gamma"], g["lam"])
    np.testing.assert_allclose(A[0], g["A"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(R[0], g["R"], rtol=0, atol=1e-15)


def test_printed_gamma(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "gamma_printed.json")))
    for case in g["cases"]:
        for T in (4.0 / 30.0, 0.133):
            gamma = oracle.gamma_from_horizon(case["horizon_s"], T)
            assert f"{gamma:.{case['digits']}f}" == case["printed"]


def _rollouts(seed, R=3, L=37, p_done=0.0):
    ro = synth.make_rollouts(R, L, seed, p_done=p_done)
    return ro["r"].astype(np.float64), ro["V"].astype(np.float64), ro["done"]


@pytest.mark.parametrize("seed", range(5))
def test_lambda0_is_td_residual(seed):
    r, V, d = _rollouts(seed, p_done=0.1)
    gamma = 0.97
    A, _ = oracle.gae(r, V, d, gamma, 0.0)
    # lambda = 0: advantage is the one-step TD residual of each step (no carry)
    for i in range(r.shape[0]):
        for t in range(r.shape[1]):
            boot = 0.0 if d[i, t] else V[i, t + 1]
            assert abs(A[i, t] - (r[i, t] + gamma * boot - V[i, t])) < 1e-13


@pytest.mark.parametrize("seed", range(5))
def test_lambda1_is_discounted_return_minus_value(seed):
    r, V, d = _rollouts(seed)
    gamma = 0.9
    L = r.shape[1]
    A, R = oracle.gae(r, V, d, gamma, 1.0)
    for i in range(r.shape[0]):
        for t in range(L):
            mc = sum(gamma ** l * r[i, t + l] for l in range(L - t)) + gamma ** (L - t) * V[i, L]
            assert abs(A[i, t] - (mc - V[i, t])) < 1e-11
            assert abs(R[i, t] - mc) < 1e-11


@pytest.mark.parametrize("seed", range(5))
def test_brute_force_double_sum_with_dones(seed):
    """A_t = sum_{l=0}^{e-t} (gamma lam)^l delta_{t+l}, stopping at the first done e >= t,
    where delta_e carries no bootstrap (P:1244 GAE definition; reading Q10)."""
    r, V, d = _rollouts(seed, R=4, L=41, p_done=0.08)
    gamma, lam = 0.99926, 0.95
    L = r.shape[1]
    A, _ = oracle.gae(r, V, d, gamma, lam)
    for i in range(r.shape[0]):
        delta = [r[i, t] + (0.0 if d[i, t] else gamma * V[i, t + 1]) - V[i, t] for t in range(L)]
        for t in range(L):
            s = 0.0
            for l in range(L - t):
                s += (gamma * lam) ** l * delta[t + l]
                if d[i, t + l]:
                    break
            assert abs(A[i, t] - s) < 1e-12


def test_done_step_is_reward_minus_value():
    r, V, d = _rollouts(7, p_done=0.0)
    d = d.copy()
    d[:, 10] = 1
    A, _ = oracle.gae(r, V, d, 0.999, 0.95)
    np.testing.assert_allclose(A[:, 10], r[:, 10] - V[:, 10], atol=1e-14)


def test_segments_to_sequences_layout():
    R_, L, T = 3, 32, 16
    a = np.arange(R_ * L).reshape(R_, L)
    s = oracle.segments_to_sequences(a, T)
    assert s.shape == (T, R_ * L // T)
    for r_ in range(R_):
        for k in range(L // T):
            for t in range(T):
                assert s[t, r_ * (L // T) + k] == a[r_, k * T + t]
