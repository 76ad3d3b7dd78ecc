"""ORACLE (test infrastructure only) -- the experience buffer of NEXT-1.

P:764 [App. Scale, Sample reuse] each optimizer GPU keeps an experience buffer; P:1249-1250
[§3.2] "Each optimizer GPU computes gradients using minibatches sampled randomly from its
experience buffer"; P:908 32 gradient steps per iteration; P:1256 a new version is
published every 32 gradient steps.  Reading Q19: uniform sampling with replacement, by the
counter-based generator idx[i] = splitmix64(seed + (step << 32) + i) mod capacity (Steele,
Lea & Flood 2014), written out here independently of the CUDA path.
"""
import numpy as np

M64 = (1 << 64) - 1


def splitmix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def sample_indices(capacity: int, B: int, seed: int, step: int) -> np.ndarray:
    """Minibatch of B sequence slots, uniform with replacement."""
    base = (seed + (step << 32)) & M64
    return np.array([splitmix64((base + i) & M64) % capacity for i in range(B)], np.int64)


def gather(buf: dict, idx) -> dict:
    """Sequence-major buffer arrays [cap][T][...] / [cap][...] -> minibatch, time-major
    [T][B][...] (x, act, head_on, avail, logp_old, adv, ret, valid) and [B][...] (h0, c0)."""
    idx = np.asarray(idx)
    out = {}
    for k, v in buf.items():
        if v is None:
            continue
        sel = np.asarray(v)[idx]
        out[k] = sel if k in ("h0", "c0") else np.swapaxes(sel, 0, 1)
    return out
