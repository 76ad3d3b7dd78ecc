"""ORACLE (test infrastructure only) -- Adam with the paper's per-parameter clip.

P:1254 [§3.2] "We apply the Adam optimizer [kingma2014adam]"; "Gradients are
additionally clipped per parameter to be within between +-5 sqrt(v) where v is the
running estimate of the second moment of the (unclipped) gradient."
P:917-919 [Table hyperparams] lr 5e-5, beta1 0.9, beta2 0.999.
Readings: DESIGN Q3 (v updated first from the unclipped g, raw v, m takes the
clipped g) and Q4 (eps on raw sqrt(v) with the bias factor folded into alpha_t).
"""
import math

import numpy as np


def adam_clip(theta, g, m, v, t, lr, beta1=0.9, beta2=0.999, eps=1e-8, clip_sigma=5.0):
    """DESIGN O10.  Returns new (theta, m, v); t >= 1 is the step number.

        v      <- beta2 v + (1 - beta2) g^2
        g_c     = clamp(g, -clip_sigma sqrt(v), +clip_sigma sqrt(v))   (off if 0 or inf)
        m      <- beta1 m + (1 - beta1) g_c
        alpha_t = lr sqrt(1 - beta2^t) / (1 - beta1^t)
        theta  <- theta - alpha_t m / (sqrt(v) + eps)
    """
    assert t >= 1
    theta = np.asarray(theta, np.float64)
    g = np.asarray(g, np.float64)
    m = np.asarray(m, np.float64)
    v = np.asarray(v, np.float64)
    v = beta2 * v + (1.0 - beta2) * g * g
    if clip_sigma and math.isfinite(clip_sigma):
        bound = clip_sigma * np.sqrt(v)
        g_c = np.minimum(np.maximum(g, -bound), bound)
    else:
        g_c = g
    m = beta1 * m + (1.0 - beta1) * g_c
    alpha_t = lr * math.sqrt(1.0 - beta2 ** t) / (1.0 - beta1 ** t)
    theta = theta - alpha_t * m / (np.sqrt(v) + eps)
    return theta, m, v
