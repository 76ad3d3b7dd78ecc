"""Pins for oracle.adam_clip: textbook Adam (torch.optim.Adam), hand-evaluated steps,
the +-5 sqrt(v) clip window and lr = 0."""
import math

import numpy as np
import torch

import oracle


def test_no_clip_is_textbook_adam():
    """clip off == torch.optim.Adam.  eps = 0 makes the two eps placements identical
    (Kingma & Ba §2 efficient form vs bias-corrected form); g is never zero here."""
    rng = np.random.default_rng(0)
    n = 50
    theta0 = rng.standard_normal(n)
    p = torch.nn.Parameter(torch.from_numpy(theta0.copy()))
    opt = torch.optim.Adam([p], lr=1e-2, betas=(0.9, 0.999), eps=0.0)
    theta, m, v = theta0.copy(), np.zeros(n), np.zeros(n)
    for t in range(1, 8):
        g = rng.standard_normal(n) + 0.1
        p.grad = torch.from_numpy(g.copy())
        opt.step()
        theta, m, v = oracle.adam_clip(theta, g, m, v, t, 1e-2, eps=0.0, clip_sigma=math.inf)
        np.testing.assert_allclose(theta, p.detach().numpy(), rtol=0, atol=1e-13)


def test_first_step_values():
    # m=v=0, g=1, lr=1e-3 -> delta = -1e-3 (clip off)
    th, m, v = oracle.adam_clip(np.zeros(1), np.ones(1), np.zeros(1), np.zeros(1), 1, 1e-3,
                                clip_sigma=0.0)
    # exactly -1e-3 * sqrt(v) / (sqrt(v) + eps) with sqrt(v) = sqrt(1e-3)
    assert abs(th[0] + 1e-3 * math.sqrt(1e-3) / (math.sqrt(1e-3) + 1e-8)) < 1e-16
    assert abs(th[0] + 1e-3) < 1e-9
    # clip 5: v = 1e-3, bound 5 sqrt(1e-3) = 0.158114 -> g_c = 0.158114, m = 0.0158114,
    # alpha = 1e-3 sqrt(1e-3)/0.1, delta = -alpha m / sqrt(v) = -1.58114e-4
    th, m, v = oracle.adam_clip(np.zeros(1), np.ones(1), np.zeros(1), np.zeros(1), 1, 1e-3,
                                clip_sigma=5.0)
    assert abs(v[0] - 1e-3) < 1e-18
    assert abs(m[0] - 0.1 * 5 * math.sqrt(1e-3)) < 1e-15
    assert abs(th[0] + 1.5811388e-4) < 1e-10 + 1e-12


def test_clip_bound_uses_updated_v():
    # post-update v = 0.04 and raw g = 3 -> clipped g = 5 * 0.2 = 1
    v_prev = (0.04 - 0.001 * 9.0) / 0.999
    th, m, v = oracle.adam_clip(np.zeros(1), np.array([3.0]), np.zeros(1), np.array([v_prev]), 10,
                                1e-3)
    assert abs(v[0] - 0.04) < 1e-15
    assert abs(m[0] - 0.1 * 1.0) < 1e-15


def test_constant_gradient_clip_window():
    """Constant g: v_t = (1 - 0.999^t) g^2, so 5 sqrt(v_t) < |g| iff t <= 40."""
    theta, m, v = np.zeros(1), np.zeros(1), np.zeros(1)
    for t in range(1, 46):
        m_prev = m.copy()
        theta, m, v = oracle.adam_clip(theta, np.ones(1), m, v, t, 1e-3)
        unclipped_m = 0.9 * m_prev + 0.1 * 1.0
        clipped = abs(m[0] - unclipped_m[0]) > 1e-15
        assert clipped == (t <= 40), t


def test_lr_zero_keeps_params_moments_advance():
    # P:2038 (surgery warm restart with lr = 0): parameters frozen, statistics move
    rng = np.random.default_rng(1)
    th0 = rng.standard_normal(10)
    th, m, v = th0.copy(), np.zeros(10), np.zeros(10)
    for t in range(1, 4):
        th, m, v = oracle.adam_clip(th, rng.standard_normal(10), m, v, t, 0.0)
    assert np.array_equal(th, th0)
    assert np.all(v > 0) and np.all(m != 0)


def test_eps_placement_where_it_matters():
    """DESIGN Q4 pinned by a case where eps dominates: first step, g = 1e-8, m = v = 0,
    lr = 1e-3, clip off.  Hand evaluation (eps = 1e-8 on the RAW sqrt(v), bias factors
    folded into alpha_t, Kingma & Ba §2 last paragraph / TF1's AdamOptimizer):
        v = 0.001 * 1e-16 = 1e-19,  sqrt(v) = 3.16227766e-10,  m = 0.1 * 1e-8 = 1e-9,
        alpha_1 = 1e-3 * sqrt(0.001) / 0.1 = 3.16227766e-4,
        delta = -3.16227766e-4 * 1e-9 / (3.16227766e-10 + 1e-8) = -3.0653430e-5.
    The other placement (eps on the bias-corrected sqrt(v_hat) = 1e-8, m_hat = 1e-8, as in
    torch.optim.Adam) gives -1e-3 * 1e-8 / 2e-8 = -5.0e-4: 16x larger, so either a moved eps
    or a dropped bias factor fails here."""
    th, m, v = oracle.adam_clip(np.zeros(1), np.array([1e-8]), np.zeros(1), np.zeros(1), 1,
                                1e-3, clip_sigma=0.0)
    assert abs(th[0] - (-3.0653430e-5)) < 1e-12
    assert abs(th[0] - (-5.0e-4)) > 1e-4
    # and torch.optim.Adam (eps on sqrt(v_hat)) really is the other reading
    p = torch.nn.Parameter(torch.zeros(1, dtype=torch.float64))
    opt = torch.optim.Adam([p], lr=1e-3, betas=(0.9, 0.999), eps=1e-8)
    p.grad = torch.tensor([1e-8], dtype=torch.float64)
    opt.step()
    assert abs(p.item() - (-5.0e-4)) < 1e-12
