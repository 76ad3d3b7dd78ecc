"""Pins for oracle.lstm: closed forms, torch.nn.LSTM (fp64, CPU) and finite differences."""
import numpy as np
import pytest
import torch

import oracle


def _params(rng, H, D, scale=0.5):
    return (scale * rng.standard_normal((4 * H, D)), scale * rng.standard_normal((4 * H, H)),
            scale * rng.standard_normal(4 * H))


def test_zero_params_closed_form():
    """All parameters zero: every gate is sigma(0)=1/2 and g = tanh(0) = 0, so
    c_t = c_{t-1}/2 and h_t = tanh(c_t)/2."""
    rng = np.random.default_rng(0)
    T, B, H, D = 5, 3, 4, 6
    x = rng.standard_normal((T, B, D))
    h0 = rng.standard_normal((B, H))
    c0 = rng.standard_normal((B, H))
    out = oracle.lstm_forward(np.zeros((4 * H, D)), np.zeros((4 * H, H)), np.zeros(4 * H), x, h0, c0)
    for t in range(T):
        ct = c0 * 0.5 ** (t + 1)
        np.testing.assert_allclose(out["c"][t], ct, atol=1e-15)
        np.testing.assert_allclose(out["h"][t], 0.5 * np.tanh(ct), atol=1e-15)


@pytest.mark.parametrize("seed", range(3))
def test_matches_torch_lstm_forward_and_grads(seed):
    rng = np.random.default_rng(seed)
    T, B, H, D = 6, 3, 5, 7
    Wx, Wh, b = _params(rng, H, D)
    x = rng.standard_normal((T, B, D))
    h0 = 0.5 * rng.standard_normal((B, H))
    c0 = rng.standard_normal((B, H))
    G = rng.standard_normal((T, B, H))  # loss = sum(G * h)

    lstm = torch.nn.LSTM(D, H, num_layers=1, bias=True).double()
    with torch.no_grad():
        lstm.weight_ih_l0.copy_(torch.from_numpy(Wx))
        lstm.weight_hh_l0.copy_(torch.from_numpy(Wh))
        lstm.bias_ih_l0.copy_(torch.from_numpy(b))
        lstm.bias_hh_l0.zero_()
    xt = torch.from_numpy(x).requires_grad_(True)
    hs, (hT, cT) = lstm(xt, (torch.from_numpy(h0)[None], torch.from_numpy(c0)[None]))
    (hs * torch.from_numpy(G)).sum().backward()

    out = oracle.lstm_forward(Wx, Wh, b, x, h0, c0)
    np.testing.assert_allclose(out["h"], hs.detach().numpy(), rtol=0, atol=1e-13)
    np.testing.assert_allclose(out["c"][-1], cT[0].detach().numpy(), rtol=0, atol=1e-13)
    dWx, dWh, db, dz = oracle.lstm_backward(out, G)
    # NEXT-4: the input gradient dL/dx_t = dz_t W_x equals autograd's x.grad
    np.testing.assert_allclose(oracle.lstm_input_grad(Wx, dz), xt.grad.numpy(), rtol=0, atol=1e-12)
    np.testing.assert_allclose(dWx, lstm.weight_ih_l0.grad.numpy(), rtol=0, atol=1e-12)
    np.testing.assert_allclose(dWh, lstm.weight_hh_l0.grad.numpy(), rtol=0, atol=1e-12)
    np.testing.assert_allclose(db, lstm.bias_ih_l0.grad.numpy(), rtol=0, atol=1e-12)
    # torch's single-bias-equivalent: bias_hh gets the same gradient as bias_ih
    np.testing.assert_allclose(db, lstm.bias_hh_l0.grad.numpy(), rtol=0, atol=1e-12)


def test_finite_differences():
    rng = np.random.default_rng(11)
    T, B, H, D = 4, 2, 3, 4
    Wx, Wh, b = _params(rng, H, D)
    x = rng.standard_normal((T, B, D))
    h0 = 0.3 * rng.standard_normal((B, H))
    c0 = rng.standard_normal((B, H))
    G = rng.standard_normal((T, B, H))

    def L(Wx_, Wh_, b_):
        return float(np.sum(G * oracle.lstm_forward(Wx_, Wh_, b_, x, h0, c0)["h"]))

    dWx, dWh, db, _ = oracle.lstm_backward(oracle.lstm_forward(Wx, Wh, b, x, h0, c0), G)
    eps = 1e-6
    for name, P, dP in (("Wx", Wx, dWx), ("Wh", Wh, dWh), ("b", b, db)):
        for idx in np.ndindex(P.shape):
            Pp, Pm = P.copy(), P.copy()
            Pp[idx] += eps
            Pm[idx] -= eps
            args_p = dict(Wx_=Wx, Wh_=Wh, b_=b)
            args_m = dict(Wx_=Wx, Wh_=Wh, b_=b)
            args_p[name + "_"] = Pp
            args_m[name + "_"] = Pm
            fd = (L(**args_p) - L(**args_m)) / (2 * eps)
            assert abs(fd - dP[idx]) <= 1e-6 * max(1.0, abs(fd)), (name, idx, fd, dP[idx])


def test_truncation_no_grad_through_h0():
    """TBPTT: weight gradients do not depend on any gradient w.r.t. h0/c0 --
    the oracle returns none; with T=1 dW_h = dz^T h0 exactly (one cell, closed form)."""
    rng = np.random.default_rng(3)
    H, D, B = 3, 2, 2
    Wx, Wh, b = _params(rng, H, D)
    x = rng.standard_normal((1, B, D))
    h0 = rng.standard_normal((B, H))
    c0 = rng.standard_normal((B, H))
    G = rng.standard_normal((1, B, H))
    out = oracle.lstm_forward(Wx, Wh, b, x, h0, c0)
    dWx, dWh, db, dz = oracle.lstm_backward(out, G)
    np.testing.assert_allclose(dWh, dz[0].T @ h0, atol=1e-14)
    np.testing.assert_allclose(dWx, dz[0].T @ x[0], atol=1e-14)
