"""a9 + a10 at world 2, 4 and 8 on ONE GPU ("Gradients are averaged across the pool
using NCCL2 allreduce before being synchronously applied"; P:1254-1255 Adam with the
+-5 sqrt(v) clip).

`ppo_test_dp_adam` runs the fused exchange kernel of `ppo_dp_adam_step` (reduce-scatter of
the gradients, Adam on the owner's shard, all-gather of the bf16 shadow -- or of theta on the
fp32 path) once per VIRTUAL rank on this device, with the same shard bounds, peer-pointer
table, rank-order sum and 1/N scale as on N GPUs.  Reference: `oracle.dp_average` over the
N gradients, then `oracle.adam_clip` on the average (DESIGN Q15: average first, then clip).

Inputs.  Each rank's gradient element is k_j * 2^e with an integer |k_j| < 2^11 shared
exponent e per element (e in [-34, -4]), so the rank-order fp32 sum and the power-of-two
scale 1/N are EXACT in binary32: the average the kernel forms equals the oracle's, and the
comparison isolates the Adam arithmetic at the 1e-6 term-scale bar of test_adam_parity
(ranks with opposite signs make averages that cancel to tiny values or exactly zero).
Sizes cover n % 4 != 0 (the scalar tail), n % 64 != 0 (a ragged last shard) and n so small
that the last ranks own empty shards.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from gpu_util import dev

pytestmark = pytest.mark.gpu

LR, B1, B2, EPS = 5e-5, 0.9, 0.999, 1e-8


@pytest.fixture(scope="module")
def L():
    from paper_1912_06680_b200 import _lib
    return _lib


def exact_grads(rng, world, n):
    e = rng.integers(-34, -4, n).astype(np.float64)
    k = rng.integers(-(1 << 11) + 1, 1 << 11, (world, n)).astype(np.float64)
    # a share of elements where the ranks cancel exactly, and some with one rank only
    cancel = rng.random(n) < 0.02
    if world > 1:
        k[1, cancel] = -k[0, cancel]
        k[2:, cancel] = 0
    g = (k * np.exp2(e)).astype(np.float32)
    assert np.array_equal(g.astype(np.float64), k * np.exp2(e))     # representable
    return g


def shard_bounds(L, n, world):
    sh = L.dp_shard(n, world)
    return sh, [(min(n, r * sh), min(n, (r + 1) * sh)) for r in range(world)]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("n", [100, 1573, (1 << 16) + 5, 1000003])
@pytest.mark.parametrize("shadow", [True, False], ids=["bf16", "fp32"])
@pytest.mark.parametrize("staged", [False, True], ids=["pull", "push"])
def test_dp_adam_world_vs_oracle(L, world, n, shadow, staged):
    if staged and world == 1:
        pytest.skip("push mode needs world > 1")
    t, clip = 3, 5.0
    rng = np.random.default_rng(1000 * world + n % 997 + 7 * shadow + 3 * staged)
    g = exact_grads(rng, world, n)
    p0 = rng.standard_normal(n).astype(np.float32)
    m0 = (1e-6 * rng.standard_normal(n)).astype(np.float32)
    v0 = (np.abs(rng.standard_normal(n)) * 1e-12).astype(np.float32)

    # oracle: a9 then a10 in fp64 (O9, O10)
    gbar = oracle.dp_average([{"g": g[j].astype(np.float64)} for j in range(world)])["g"]
    pr, mr, vr = oracle.adam_clip(p0, gbar, m0, v0, t, LR, B1, B2, EPS, clip)

    G = [dev(g[j]) for j in range(world)]
    P = [dev(p0) for _ in range(world)]
    M = [dev(m0) for _ in range(world)]
    V = [dev(v0) for _ in range(world)]
    S = [torch.full((n,), float("nan"), dtype=torch.bfloat16, device="cuda")
         for _ in range(world)] if shadow else None
    sh, bounds = shard_bounds(L, n, world)
    ST = None
    if staged:   # what every rank's lstm_bptt_bwd_dp delivers: slot i = rank i's shard grads
        ST = []
        for (lo, hi) in bounds:
            st = torch.full((world * sh,), float("nan"), device="cuda")
            for i in range(world):
                st[i * sh:i * sh + (hi - lo)] = G[i][lo:hi]
            ST.append(st)
    L.test_dp_adam(G, P, S, M, V, t, LR, B1, B2, EPS, clip, stage=ST)
    torch.cuda.synchronize()

    # reassemble the sharded results: owner r's shard of theta (bf16 path) / m / v
    th = np.empty(n, np.float64)
    mm = np.empty(n, np.float64)
    vv = np.empty(n, np.float64)
    for r, (lo, hi) in enumerate(bounds):
        pr_r, m_r, v_r = (x.cpu().numpy() for x in (P[r], M[r], V[r]))
        th[lo:hi], mm[lo:hi], vv[lo:hi] = pr_r[lo:hi], m_r[lo:hi], v_r[lo:hi]
        out = np.ones(n, bool)
        out[lo:hi] = False                       # outside the shard: untouched
        assert np.array_equal(m_r[out], m0[out]) and np.array_equal(v_r[out], v0[out]), r
        if shadow:
            assert np.array_equal(pr_r[out], p0[out]), r
    # the per-element fp32 rounding scale of each output's terms (as test_adam_parity)
    ga = np.abs(gbar)
    gc_mag = np.minimum(ga, clip * np.sqrt(vr))
    scale_v = B2 * np.abs(v0) + (1 - B2) * ga * ga
    scale_m = B1 * np.abs(m0) + (1 - B1) * gc_mag
    scale_p = np.abs(p0) + np.abs(pr - p0)
    for name, got, ref, sc in (("theta", th, pr, scale_p), ("m", mm, mr, scale_m),
                               ("v", vv, vr, scale_v)):
        rel = np.abs(got - ref) / (sc + 1e-30)
        assert rel.max() <= 1e-6, (name, float(rel.max()))
    d_got, d_ref = th - p0, pr - p0
    assert np.abs(d_got - d_ref).max() <= 1e-6 * np.abs(d_ref).max() + 2 ** -23 * np.abs(p0).max()
    assert (np.abs(d_ref) > 0).mean() > 0.9            # the update moved most of theta
    th32 = torch.from_numpy(th.astype(np.float32)).cuda()
    if shadow:   # the all-gathered shadow: every rank's copy complete, RNE of theta, identical
        for j in range(world):
            assert torch.equal(S[j], th32.bfloat16()), j
    else:        # fp32 path: theta itself all-gathered into every rank
        for j in range(world):
            assert torch.equal(P[j], th32), j
    # same bits as the single-GPU adam_step on the (exact) average
    Pa, Ma, Va = dev(p0), dev(m0), dev(v0)
    L.adam_step(Pa, None, dev(gbar.astype(np.float32)), Ma, Va, t, LR, B1, B2, EPS, clip)
    torch.cuda.synchronize()
    assert torch.equal(Pa, th32) and torch.equal(Ma.cpu().double(), torch.from_numpy(mm))
    assert torch.equal(Va.cpu().double(), torch.from_numpy(vv))


@pytest.mark.parametrize("world", [2, 8])
def test_dp_adam_world_identical_grads_equal_shard(L, world):
    """O9 special case: N identical shards average to the shard itself, so the fused update
    at world N equals adam_step at world 1 bit for bit.  The gradients carry <= 16
    significant bits, so the rank-order partial sums g, 2g, ..., 8g are exact in binary32
    and the scale 1/N (a power of two) is exact too."""
    n = 64 * 1000 + 3
    rng = np.random.default_rng(world)
    g = rng.standard_normal(n) * np.exp(rng.uniform(-6, 2, n))
    e = np.floor(np.log2(np.abs(g)))
    g = (np.round(g * np.exp2(15 - e)) * np.exp2(e - 15)).astype(np.float32)   # 16-bit mantissas
    p0 = rng.standard_normal(n).astype(np.float32)
    z = np.zeros(n, np.float32)
    for t in (1, 2):
        G = [dev(g) for _ in range(world)]
        P, M, V = [dev(p0) for _ in range(world)], [dev(z) for _ in range(world)], [dev(z) for _ in range(world)]
        S = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(world)]
        L.test_dp_adam(G, P, S, M, V, t, LR, B1, B2, EPS, 5.0)
        Pa, Ma, Va = dev(p0), dev(z), dev(z)
        Sa = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        L.adam_step(Pa, Sa, dev(g), Ma, Va, t, LR, B1, B2, EPS, 5.0)
        torch.cuda.synchronize()
        # sum of N equal fp32 values then 1/N: exact for N a power of two
        for j in range(world):
            assert torch.equal(S[j], Sa)
        _, bounds = shard_bounds(L, n, world)
        for r, (lo, hi) in enumerate(bounds):
            assert torch.equal(P[r][lo:hi], Pa[lo:hi]) and torch.equal(M[r][lo:hi], Ma[lo:hi])


def test_dp_adam_hook_errors(L):
    x = torch.zeros(64, device="cuda")
    with pytest.raises(L.PPOError):
        L.test_dp_adam([x] * 9, [x] * 9, None, [x] * 9, [x] * 9, 1, LR, B1, B2, EPS, 5.0)
    with pytest.raises(L.PPOError):
        L.test_dp_adam([x] * 2, [x] * 2, None, [x] * 2, [x] * 2, 0, LR, B1, B2, EPS, 5.0)
    with pytest.raises(L.PPOError):   # misaligned
        y = torch.zeros(80, device="cuda")[1:65]
        L.test_dp_adam([y] * 2, [y] * 2, None, [y] * 2, [y] * 2, 1, LR, B1, B2, EPS, 5.0)
    assert math.isfinite(float(x.sum()))
