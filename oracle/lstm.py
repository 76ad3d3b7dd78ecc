"""ORACLE (test infrastructure only) -- the single-layer LSTM and its truncated BPTT.

P:1210 [§3.1] "a single-layer 4096-unit LSTM [gers1999learning]": the forget-gate LSTM
without peepholes.  P:1254 [§3.2] "truncated backpropagation through time over
samples of 16 timesteps".  P:1202 each hero replica has its own hidden state.
Canonical layout: z = x W_x^T + h W_h^T + b with gate blocks [i; f; g; o] (DESIGN Q14).
"""
import numpy as np


def _sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def lstm_forward(Wx, Wh, b, x, h0, c0):
    """DESIGN O4.  x [T][B][D], h0/c0 [B][H]; returns dict with
    h [T][B][H], c [T][B][H] and the per-step gates for backward.

    for t = 0 .. T-1:
        z = x_t W_x^T + h_{t-1} W_h^T + b
        i = sigma(z_i), f = sigma(z_f), g = tanh(z_g), o = sigma(z_o)
        c_t = f * c_{t-1} + i * g
        h_t = o * tanh(c_t)
    """
    Wx = np.asarray(Wx, np.float64)
    Wh = np.asarray(Wh, np.float64)
    b = np.asarray(b, np.float64)
    x = np.asarray(x, np.float64)
    h = np.asarray(h0, np.float64)
    c = np.asarray(c0, np.float64)
    T, B, _ = x.shape
    H = Wh.shape[1]
    hs, cs, gates = [], [], []
    for t in range(T):
        z = x[t] @ Wx.T + h @ Wh.T + b
        i = _sigmoid(z[:, 0 * H:1 * H])
        f = _sigmoid(z[:, 1 * H:2 * H])
        g = np.tanh(z[:, 2 * H:3 * H])
        o = _sigmoid(z[:, 3 * H:4 * H])
        c = f * c + i * g
        h = o * np.tanh(c)
        hs.append(h)
        cs.append(c)
        gates.append((i, f, g, o))
    return dict(x=x, h0=np.asarray(h0, np.float64), c0=np.asarray(c0, np.float64),
                h=np.stack(hs), c=np.stack(cs), gates=gates, Wx=Wx, Wh=Wh)


def lstm_backward(cache, dh_out):
    """DESIGN O8.  dh_out [T][B][H] = dL/dh_t from the heads.  Truncated BPTT:
    no gradient flows into h0 / c0.

    for t = T-1 .. 0:
        dh      = dh_out_t + dh_rec
        dc      = dc_next + dh * o * (1 - tanh(c_t)^2)
        do = dh * tanh(c_t);  di = dc * g;  dg = dc * i;  df = dc * c_{t-1}
        dc_next = dc * f
        dz      = [di i(1-i), df f(1-f), dg (1-g^2), do o(1-o)]
        dh_rec  = dz W_h
        dW_x += dz^T x_t;  dW_h += dz^T h_{t-1};  db += sum_b dz
    Returns (dWx, dWh, db, dz [T][B][4H]).
    """
    x, h, c = cache["x"], cache["h"], cache["c"]
    Wx, Wh = cache["Wx"], cache["Wh"]
    T, B, _ = x.shape
    H = Wh.shape[1]
    dWx = np.zeros_like(Wx)
    dWh = np.zeros_like(Wh)
    db = np.zeros(4 * H)
    dh_rec = np.zeros((B, H))
    dc_next = np.zeros((B, H))
    dzs = np.zeros((T, B, 4 * H))
    for t in reversed(range(T)):
        i, f, g, o = cache["gates"][t]
        c_prev = c[t - 1] if t > 0 else cache["c0"]
        h_prev = h[t - 1] if t > 0 else cache["h0"]
        tc = np.tanh(c[t])
        dh = dh_out[t] + dh_rec
        dc = dc_next + dh * o * (1.0 - tc * tc)
        do = dh * tc
        di = dc * g
        dg = dc * i
        df = dc * c_prev
        dc_next = dc * f
        dz = np.concatenate([di * i * (1 - i), df * f * (1 - f),
                             dg * (1 - g * g), do * o * (1 - o)], axis=1)
        dzs[t] = dz
        dh_rec = dz @ Wh
        dWx += dz.T @ x[t]
        dWh += dz.T @ h_prev
        db += dz.sum(axis=0)
    return dWx, dWh, db, dzs


def lstm_input_grad(Wx, dz):
    """NEXT-4, the dX output for upstream observation processing (P:1204-1212 [§3.1]: the
    LSTM input is the output of the observation-processing network, which is trained
    through it): dL/dx_t = dz_t W_x for every t.  dz [T][B][4H] from lstm_backward."""
    return np.asarray(dz, np.float64) @ np.asarray(Wx, np.float64)
