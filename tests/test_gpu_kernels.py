"""Isolated-kernel parity on the GPU (each ABI call fed identical inputs vs the oracle, or vs
plain PyTorch fp32 for the GEMM core)."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import dev, elementwise_ok

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1912_06680_b200 import _lib
    return _lib


# ------------------------------------------------------------------ tcgen05 GEMM core
@pytest.mark.parametrize("mode,M,N,K", [
    (0, 128, 256, 64), (0, 300, 520, 200), (0, 1000, 16384 // 8, 1024),
    (1, 256, 512, 192), (1, 77, 264, 1000),
    (3, 384, 768, 448), (3, 136, 320, 72),
    (4, 300, 656, 4160), (4, 33, 100, 64),
    # CTA-pair (cta_group::2) kernel, 256x256 tiles
    (8, 256, 256, 64), (8, 300, 520, 200), (8, 1000, 2048, 1024),
    (9, 512, 512, 192), (9, 77, 264, 1000),
    (11, 384, 768, 448), (11, 136, 320, 72), (11, 2048, 1024, 4096),
    # CTA pair with 512-row tiles (two MMAs per K step), MN-major operands (weight gradient)
    (27, 512, 256, 64), (27, 600, 520, 200), (27, 2048, 1024, 4096),
    # CTA pair with N=224 tiles (heads), K-major
    (40, 300, 656, 4160), (40, 1000, 448, 192),
])
def test_tc_gemm_vs_torch(L, mode, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    a_mn, b_mn = bool(mode & 2), bool(mode & 1)  # bit2: N=224, bit3: CTA pair, bit4: 512 rows
    A = torch.randn((K, M) if a_mn else (M, K), generator=g, device="cuda").bfloat16()
    B = torch.randn((K, N) if b_mn else (N, K), generator=g, device="cuda").bfloat16()
    C = torch.full((M, N), float("nan"), device="cuda")
    L.test_tc_gemm(mode, A, B, C, M, N, K)
    torch.cuda.synchronize()
    Af = (A.t() if a_mn else A).float()
    Bf = (B if b_mn else B.t()).float()
    ref = (Af.double() @ Bf.double()).float()
    err = ((C - ref).abs().max() / ref.abs().max()).item()
    assert not torch.isnan(C).any()
    assert err < 1e-5, err


# ------------------------------------------------------------------ GAE
@pytest.mark.parametrize("R,Lr,seq_T,p_done", [
    (2, 256, 16, 0.01), (2400, 256, 16, 1 / 20000), (3, 1350, 0, 0.002), (5, 1, 0, 0.5),
    # row starts off the 8-step grid: shifted first windows, window rounding (L % 8 != 0)
    (11, 1350, 0, 0.01), (13, 257, 0, 0.01), (9, 263, 0, 0.02), (17, 7, 0, 0.1),
    # 600 <= R < 4736 streams: 16-step lane chunks (512-step windows)
    (700, 3000, 0, 1e-3), (1000, 2112, 16, 1e-3), (1000, 300, 0, 0.05), (2100, 520, 0, 0.01),
    (1, 6300, 0, 0.0), (7, 300, 0, 0.05), (4, 512, 16, 0.0),
    # long rollouts: chunk-parallel look-back kernel (chunks of 8192 steps), ragged tails
    (1, 20000, 0, 1 / 20000), (3, 100001, 0, 1e-4), (2, 8193, 0, 0.0), (5, 40960, 16, 0.001),
    (1, 1000000, 0, 1e-5), (16384, 9000, 0, 1e-4),
])
def test_gae_parity(L, R, Lr, seq_T, p_done):
    ro = synth.make_rollouts(R, Lr, seed=R + Lr, p_done=p_done)
    gamma = float(np.float32(oracle.gamma_from_horizon(180.0)))
    lam = float(np.float32(0.95))
    A, Rt = oracle.gae(ro["r"], ro["V"], ro["done"], gamma, lam)
    if seq_T:
        A = oracle.segments_to_sequences(A, seq_T)
        Rt = oracle.segments_to_sequences(Rt, seq_T)
    adv = torch.full(A.shape, float("nan"), device="cuda")
    ret = torch.full(A.shape, float("nan"), device="cuda")
    nb = L.gae_scratch_bytes(R, Lr)
    scratch = torch.empty(nb, dtype=torch.uint8, device="cuda") if nb else None
    L.ppo_gae(dev(ro["r"]), dev(ro["V"]), dev(ro["done"]), gamma, lam, adv, ret, seq_T=seq_T,
              scratch=scratch)
    torch.cuda.synchronize()
    ok, worst = elementwise_ok(adv.cpu().numpy(), A, 1e-5)
    assert ok, worst
    ok, worst = elementwise_ok(ret.cpu().numpy(), Rt, 1e-5)
    assert ok, worst


def test_gae_misaligned_bases(L):
    """Buffers that start off the 32-byte grid take the scalar path (same results)."""
    R, Lr = 6, 1000
    ro = synth.make_rollouts(R, Lr, seed=3, p_done=0.01)
    gamma = float(np.float32(oracle.gamma_from_horizon(180.0)))
    lam = float(np.float32(0.95))
    A, Rt = oracle.gae(ro["r"], ro["V"], ro["done"], gamma, lam)
    def shifted(a, dtype):
        t = torch.from_numpy(np.ascontiguousarray(a)).to("cuda")
        buf = torch.empty(t.numel() + 1, dtype=t.dtype, device="cuda")
        v = buf[1:].view(t.shape)
        v.copy_(t)
        return v
    adv = torch.empty(R * Lr + 1, device="cuda")[1:].view(R, Lr)
    ret = torch.empty(R * Lr + 1, device="cuda")[1:].view(R, Lr)
    L.ppo_gae(shifted(ro["r"], None), shifted(ro["V"], None), shifted(ro["done"], None), gamma,
              lam, adv, ret)
    torch.cuda.synchronize()
    ok, worst = elementwise_ok(adv.cpu().numpy(), A, 1e-5)
    assert ok, worst
    ok, worst = elementwise_ok(ret.cpu().numpy(), Rt, 1e-5)
    assert ok, worst


def test_gae_lambda_edge_cases(L):
    """lambda = 0 -> TD residual; gamma = lambda = 1 with no dones -> return-to-go minus V."""
    ro = synth.make_rollouts(3, 64, seed=9, p_done=0.0)
    for gamma, lam in ((0.99, 0.0), (1.0, 1.0)):
        A, _ = oracle.gae(ro["r"], ro["V"], ro["done"], gamma, lam)
        adv = torch.empty(A.shape, device="cuda")
        ret = torch.empty(A.shape, device="cuda")
        L.ppo_gae(dev(ro["r"]), dev(ro["V"]), dev(ro["done"]), gamma, lam, adv, ret)
        torch.cuda.synchronize()
        ok, worst = elementwise_ok(adv.cpu().numpy(), A, 1e-5)
        assert ok, (gamma, lam, worst)


# ------------------------------------------------------------------ PPO loss
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
# B = 643 and 4,000: several rows per warp of the persistent loss kernel (its buffer
# rotation, one-row-ahead metadata and bulk stores) with a ragged last run
@pytest.mark.parametrize("seed,pad,B", [(0, 0.0, 40), (1, 0.5, 40), (2, 0.0, 40), (3, 0.3, 643),
                                        (4, 0.1, 4000)])
def test_loss_parity(L, precision, seed, pad, B):
    T = 16
    cfg = synth.Config(H=64, D=64, B=B, T=T)
    s = synth.make_sequences(cfg, seed, pad_frac=pad)
    N = T * B
    Y = synth.make_logits(N, cfg.A, seed, scale=1.5)
    rng = np.random.default_rng(seed)
    adv = rng.standard_normal(N).astype(np.float32)
    ret = rng.standard_normal(N).astype(np.float32)
    act, on, av, valid = (s[k].reshape(N, -1) for k in ("act", "head_on", "avail", "valid"))
    valid = valid.reshape(N)
    lp0 = oracle.ppo_loss(Y, act, on, av, np.zeros(N), adv, ret, None, cfg.head_sizes)[3]
    logp_old = (lp0 + s["logp_noise"].reshape(N)).astype(np.float32)
    Lref, dYref, st, lpref = oracle.ppo_loss(Y, act, on, av, logp_old, adv, ret, valid,
                                             cfg.head_sizes, 0.2, 1.0, 0.01)
    bf16 = precision == "bf16"
    dims = L.make_dims(64, 64, T, cfg.head_sizes, L.PPO_PREC_BF16 if bf16 else L.PPO_PREC_FP32)
    dout = torch.empty((N, cfg.A), device="cuda", dtype=torch.bfloat16 if bf16 else torch.float32)
    logp = torch.empty(N, device="cuda")
    stats = torch.zeros(L.PPO_STATS_BUF, device="cuda")
    L.ppo_loss_grad(dims, dev(Y), dev(act), dev(on), dev(av), dev(logp_old), dev(adv), dev(ret),
                    dev(valid), B, L.ppo_loss_cfg(0.2, 1.0, 0.01, 0.0), dout, logp, stats)
    torch.cuda.synchronize()
    ok, worst = elementwise_ok(logp.cpu().numpy(), lpref, 1e-5)
    assert ok, worst
    d = dout.float().cpu().numpy()
    if bf16:
        # bf16 storage of an fp32 result: one rounding (2^-9 relative)
        assert np.all(np.abs(d - dYref) <= 2 ** -8 * np.abs(dYref) + 1e-12)
    else:
        ok, worst = elementwise_ok(d, dYref, 1e-5)
        assert ok, worst
    # masked entries are exactly zero
    assert np.all(d[:, :30][av == 0] == 0.0)
    assert np.all(d[valid == 0] == 0.0)
    sv = stats[:8].cpu().numpy()
    check_loss_stats(sv, st, lpref, logp_old, adv, Y[:, -1], ret, valid, N)


def check_loss_stats(sv, st, lpref, logp_old, adv, V, ret, valid, denom, clip_rows=None):
    """Loss statistics vs the oracle, relative: |x - x_ref| <= 1e-5 |x_ref| + 2^-22 S, where S
    = sum_rows w |term| / denom is the scale of the terms the statistic sums (the fp32 / SFU
    lg2 rounding of each term, 2^-22 relative, is what a sum that cancels -- pg,
    approx_kl -- cannot resolve below).  clipfrac and n_valid are counts: exact."""
    w = np.asarray(valid, np.float64).reshape(-1)
    lo = np.asarray(logp_old, np.float64).reshape(-1)
    lp = np.asarray(lpref, np.float64).reshape(-1)
    rho = np.exp(lp - lo)
    s_pg = np.sum(w * np.abs(rho * np.asarray(adv, np.float64).reshape(-1))) / denom
    s_vf = np.sum(w * (np.asarray(V, np.float64) - np.asarray(ret, np.float64).reshape(-1)) ** 2) / denom
    scale = dict(pg=s_pg, vf=s_vf, ent=abs(st["ent"]), loss=s_pg + s_vf + 0.01 * abs(st["ent"]),
                 approx_kl=np.sum(w * (np.abs(lo) + np.abs(lp))) / denom)
    for i, k in enumerate(("loss", "pg", "vf", "ent", "approx_kl")):
        tol = 1e-5 * abs(st[k]) + 2.0 ** -22 * scale[k]
        assert abs(sv[i] - st[k]) <= tol, (k, float(sv[i]), st[k], tol)
    n_clip = sv[5] * denom if clip_rows is None else clip_rows
    assert round(float(sv[5]) * denom) == round(st["clipfrac"] * denom) == round(n_clip), \
        (sv[5] * denom, st["clipfrac"] * denom)
    assert sv[6] == st["n_valid"]
    assert int(sv[7]) == st["flags"] == 0


def _loss_call(L, cfg, T, B, Y, act, on, av, logp_old, adv, ret, valid, clip_eps, bf16=False):
    dims = L.make_dims(64, 64, T, cfg.head_sizes, L.PPO_PREC_BF16 if bf16 else L.PPO_PREC_FP32)
    N = T * B
    dout = torch.full((N, cfg.A), float("nan"), device="cuda",
                      dtype=torch.bfloat16 if bf16 else torch.float32)
    logp = torch.empty(N, device="cuda")
    stats = torch.zeros(L.PPO_STATS_BUF, device="cuda")
    L.ppo_loss_grad(dims, dev(Y), dev(act), dev(on), dev(av), dev(logp_old), dev(adv), dev(ret),
                    None if valid is None else dev(valid), B,
                    L.ppo_loss_cfg(clip_eps, 1.0, 0.01, 0.0), dout, logp, stats)
    torch.cuda.synchronize()
    return dout.float().cpu().numpy(), logp.cpu().numpy(), stats[:8].cpu().numpy()


def test_loss_clip_tie_exact(L):
    """DESIGN Q8 at an exact tie: clip_eps = 0 and rho = 1 exactly on every row (each side's
    logp_old is its OWN log pi -- the oracle's fp64 value, the GPU's fp32 value -- so
    exp(0) = 1 on both), hence rho A == clip(rho) A.  Ties take the unclipped branch: the
    policy gradient flows on every row and clipfrac is exactly 0 (a strict '<' would zero it)."""
    T, B = 16, 40
    cfg = synth.Config(H=64, D=64, B=B, T=T)
    s = synth.make_sequences(cfg, 21)
    N = T * B
    Y = synth.make_logits(N, cfg.A, 21, scale=1.5)
    rng = np.random.default_rng(21)
    adv = rng.standard_normal(N).astype(np.float32)
    ret = rng.standard_normal(N).astype(np.float32)
    act, on, av = (s[k].reshape(N, -1) for k in ("act", "head_on", "avail"))
    lp_o = oracle.ppo_loss(Y, act, on, av, np.zeros(N), adv, ret, None, cfg.head_sizes)[3]
    _, dYref, st, _ = oracle.ppo_loss(Y, act, on, av, lp_o, adv, ret, None, cfg.head_sizes,
                                      0.0, 1.0, 0.01)
    assert st["clipfrac"] == 0.0
    z = np.zeros(N, np.float32)
    _, lp_g, _ = _loss_call(L, cfg, T, B, Y, act, on, av, z, adv, ret, None, 0.0)
    d, lp2, sv = _loss_call(L, cfg, T, B, Y, act, on, av, lp_g, adv, ret, None, 0.0)
    assert np.array_equal(lp2, lp_g)                       # rho = exp(0) = 1 on the GPU
    assert sv[5] == 0.0, sv[5]
    ok, worst = elementwise_ok(d, dYref, 1e-5)
    assert ok, worst


@pytest.mark.parametrize("side", [+1, -1])
def test_loss_clip_edges(L, side):
    """rho placed on the clip edges 1 +- eps (logp_old = log pi - log(1 +- eps), each side
    from its own log pi).  At the edge rho is an fp32 rounding away from 1 +- eps, so the
    branch taken there is not unique: each edge row must equal the oracle's unclipped-branch
    gradient (rows with A as given) or its clipped-branch gradient (the same row with the
    policy term removed, i.e. A = 0), and clipfrac must count exactly the rows that took the
    clipped branch.  Rows 1e-3 inside / outside the edge must take the unique branch."""
    T, B = 16, 40
    eps = 0.2
    cfg = synth.Config(H=64, D=64, B=B, T=T)
    s = synth.make_sequences(cfg, 30 + side)
    N = T * B
    Y = synth.make_logits(N, cfg.A, 30 + side, scale=1.5)
    rng = np.random.default_rng(30 + side)
    # A > 0 clips above 1 + eps, A < 0 below 1 - eps: put each row's A on its edge's side
    adv = (side * np.abs(rng.standard_normal(N)) + side * 0.1).astype(np.float32)
    ret = rng.standard_normal(N).astype(np.float32)
    act, on, av = (s[k].reshape(N, -1) for k in ("act", "head_on", "avail"))
    # row kinds: 0 on the edge, 1 inside by 1e-3 (unclipped), 2 outside by 1e-3 (clipped)
    kind = np.arange(N) % 3
    target = 1.0 + side * eps + side * np.where(kind == 1, -1e-3, np.where(kind == 2, 1e-3, 0.0))
    shift = np.log(target)
    z = np.zeros(N, np.float32)
    lp_o = oracle.ppo_loss(Y, act, on, av, z, adv, ret, None, cfg.head_sizes)[3]
    lo_o = lp_o - shift
    _, dY_unc, _, _ = oracle.ppo_loss(Y, act, on, av, lo_o, adv, ret, None, cfg.head_sizes, 1e9,
                                      1.0, 0.01)            # eps = 1e9: nothing clips
    _, dY_clp, _, _ = oracle.ppo_loss(Y, act, on, av, lo_o, z, ret, None, cfg.head_sizes, eps,
                                      1.0, 0.01)            # A = 0: no policy term
    _, lp_g, _ = _loss_call(L, cfg, T, B, Y, act, on, av, z, adv, ret, None, eps)
    lo_g = (lp_g.astype(np.float64) - shift).astype(np.float32)
    d, _, sv = _loss_call(L, cfg, T, B, Y, act, on, av, lo_g, adv, ret, None, eps)

    def rows_match(ref):
        rms = np.sqrt(np.mean(ref * ref))
        return np.all(np.abs(d - ref) <= 1e-5 * (np.abs(ref) + rms), axis=1)
    unc, clp = rows_match(dY_unc), rows_match(dY_clp)
    assert not np.any(unc & clp)         # |A| >= 0.1: the two branches differ on every row
    assert np.all(unc | clp)             # every row took one of the two valid branches
    assert np.all(unc[kind == 1]) and np.all(clp[kind == 2])
    assert round(float(sv[5]) * N) == int(np.sum(clp))      # clipfrac counts those rows


def test_loss_nonfinite_flag(L):
    """PPO_STAT_FLAGS bit0 (ppo5.h): a non-finite loss on a VALID row raises it, as the
    oracle's FLAG_NONFINITE does; the same NaN on an invalid (w = 0) row does not."""
    T, B = 1, 64
    cfg = synth.Config(H=64, D=64, B=B, T=T)
    s = synth.make_sequences(cfg, 5)
    N = T * B
    act, on, av = (s[k].reshape(N, -1) for k in ("act", "head_on", "avail"))
    rng = np.random.default_rng(5)
    adv = rng.standard_normal(N).astype(np.float32)
    ret = rng.standard_normal(N).astype(np.float32)
    for bad_row_valid in (1, 0):
        Y = synth.make_logits(N, cfg.A, 5)
        Y[9, -1] = np.nan                                     # the value output of row 9
        valid = np.ones(N, np.uint8)
        valid[9] = bad_row_valid
        st = oracle.ppo_loss(Y, act, on, av, np.zeros(N), adv, ret, valid, cfg.head_sizes)[2]
        _, _, sv = _loss_call(L, cfg, T, B, Y, act, on, av, np.zeros(N, np.float32), adv, ret,
                              valid, 0.2)
        assert (int(sv[7]) & 1) == (st["flags"] & 1) == bad_row_valid, (sv[7], st["flags"])


def test_loss_flags(L):
    T, B = 1, 64
    cfg = synth.Config(H=64, D=64, B=B, T=T)
    s = synth.make_sequences(cfg, 3)
    N = T * B
    act, on, av = (s[k].reshape(N, -1) for k in ("act", "head_on", "avail"))
    av = av.copy()
    act = act.copy()
    av[5, act[5, 0]] = 0          # taken action unavailable
    act[5, 0] = 7 if av[5, 7] == 0 else act[5, 0]
    av[6, :] = 0                  # empty availability row
    Y = synth.make_logits(N, cfg.A, 1)
    dims = L.make_dims(64, 64, T, cfg.head_sizes, L.PPO_PREC_FP32)
    stats = torch.zeros(L.PPO_STATS_BUF, device="cuda")
    z = dev(np.zeros(N, np.float32))
    L.ppo_loss_grad(dims, dev(Y), dev(act), dev(on), dev(av), z, z, z, None, B,
                    L.ppo_loss_cfg(0.2, 1.0, 0.01, 0.0),
                    torch.empty((N, cfg.A), device="cuda"), None, stats)
    torch.cuda.synchronize()
    flags = int(stats[7].item())
    assert flags & 2 and flags & 4


# ------------------------------------------------------------------ Adam + clip
@pytest.mark.parametrize("n,t,clip", [(1000, 1, 5.0), (4097, 7, 5.0), (10001, 3, 0.0),
                                      (1 << 20, 50, 5.0)])
def test_adam_parity(L, n, t, clip):
    rng = np.random.default_rng(n + t)
    p = rng.standard_normal(n).astype(np.float32)
    g = (rng.standard_normal(n) * np.exp(rng.uniform(-6, 2, n))).astype(np.float32)
    m = (0.01 * rng.standard_normal(n)).astype(np.float32)
    v = (np.abs(rng.standard_normal(n)) * 1e-4).astype(np.float32) if t > 1 else np.zeros(n, np.float32)
    pr, mr, vr = oracle.adam_clip(p, g, m, v, t, 5e-5, 0.9, 0.999, 1e-8, clip if clip else math.inf)
    # per-element magnitude of the terms each output is formed from (fp32 rounding scale)
    g64 = g.astype(np.float64)
    gc_mag = np.minimum(np.abs(g64), clip * np.sqrt(vr)) if clip else np.abs(g64)
    scale_v = 0.999 * np.abs(v) + 0.001 * g64 * g64
    scale_m = 0.9 * np.abs(m) + 0.1 * gc_mag
    scale_p = np.abs(p) + np.abs(pr - p)
    P, Gt, Mt, Vt = dev(p), dev(g), dev(m), dev(v)
    P16 = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    L.adam_step(P, P16, Gt, Mt, Vt, t, 5e-5, 0.9, 0.999, 1e-8, clip)
    torch.cuda.synchronize()
    for name, got, ref, sc in (("p", P, pr, scale_p), ("m", Mt, mr, scale_m), ("v", Vt, vr, scale_v)):
        gg = got.cpu().numpy().astype(np.float64)
        rel = np.abs(gg - ref) / (sc + 1e-30)
        assert rel.max() <= 1e-6, (name, rel.max())
    # the update itself (p_new - p_old) relative to its own size
    d_got = P.cpu().numpy().astype(np.float64) - p
    d_ref = pr - p
    assert np.abs(d_got - d_ref).max() <= 1e-6 * np.abs(d_ref).max() + 2 ** -23 * np.abs(p).max()
    assert torch.equal(P16, P.bfloat16())


# ------------------------------------------------------------------ layout
def test_pack_unpack_roundtrip_bit_exact(L):
    cfg = synth.Config(H=128, D=192, B=1)
    prm = synth.make_params(cfg, 5, bo_scale=0.1)
    dims = L.make_dims(cfg.D, cfg.H, 16, cfg.head_sizes, L.PPO_PREC_FP32)
    lay = L.param_layout(dims)
    theta = torch.full((lay.n_total,), float("nan"), device="cuda")
    L.ppo_pack_params(dims, *(dev(prm[k]) for k in ("Wx", "Wh", "b", "Wo", "bo")), theta)
    outs = {k: torch.empty(v.shape, device="cuda") for k, v in prm.items()}
    L.ppo_unpack_params(dims, theta, *(outs[k] for k in ("Wx", "Wh", "b", "Wo", "bo")))
    torch.cuda.synchronize()
    th = theta.cpu().numpy()
    assert not np.isnan(th).any()
    for k in prm:
        assert np.array_equal(outs[k].cpu().numpy(), prm[k]), k
    # spot-check the documented interleave: row r -> gate (r%256)//64 of unit 64*(r//256)+r%64
    W = th[:lay.n_wxh].reshape(4 * cfg.H, lay.Kx)
    for r in (0, 63, 64, 200, 256, 511):
        gate, unit = (r % 256) // 64, 64 * (r // 256) + r % 64
        cr = gate * cfg.H + unit
        assert np.array_equal(W[r, :cfg.D], prm["Wx"][cr])
        assert np.array_equal(W[r, cfg.D:cfg.D + cfg.H], prm["Wh"][cr])
        assert W[r, cfg.D + cfg.H] == prm["b"][cr]
        assert np.all(W[r, cfg.D + cfg.H + 1:] == 0)
