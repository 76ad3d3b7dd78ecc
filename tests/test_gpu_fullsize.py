"""Parity at BASELINE.json's full size, in the launch configuration bench.py times
(H=4096, D=4032, T=16, B=38,400 sequences, bf16 tcgen05 path), on sampled outputs -- and
again at the maximum minibatch that fits 180 GB (B_max = 123,648 sequences, 170 GB,
profiles/r01_sweep_B_v3.jsonl), the largest launch the library supports on one B200, and at
the paper's minibatch size (B = 640 ~ 600, the small-B split-K backward).

The GPU runs the whole step over all 38,400 sequences.  Per-sequence quantities (GAE of a
rollout stream, the forward pass of a sequence, the loss gradient of a row) are checked one
by one against the float64 oracle.  For the weight gradients, every row outside a few sampled
sequences is masked (valid = 0): their dL/dy is exactly zero, so dW is the sum over the sampled
sequences only, which the oracle computes with the same denominator T*B.  Adam is checked on
sampled elements of the GPU's own gradient."""
import gc

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import HYPER, elementwise_ok, normwise
from oracle.step import loss_and_grads

pytestmark = pytest.mark.gpu

B_BENCH, B_MAX = 38400, 123648
# the paper's per-GPU minibatch (600) rounded up to whole 256-step rollout streams: its
# backward steps have fewer tiles than CTA pairs, so this runs the split-K backward path
B_PAPER = 640


@pytest.fixture(scope="module", params=[B_PAPER, B_BENCH, B_MAX],
                ids=["B640", "B38400", "Bmax123648"])
def run(request):
    res = _run(request.param)
    yield res
    res.clear()
    gc.collect()
    torch.cuda.empty_cache()


def _run(B_total):
    from paper_1912_06680_b200 import PPOOptimizer
    dev = "cuda"
    cfg = synth.Config(H=4096, D=4032, B=B_total)
    # sampled sequences (first, middle, last tile); rollout streams of 256 steps (16 sequences)
    SAMPLE_SEQ = (0, min(12345, B_total // 2 + 5), B_total - 1)
    SAMPLE_STREAMS = (0, min(771, B_total // 32 + 1), B_total // 16 - 1)
    T, B, H, D = cfg.T, cfg.B, cfg.H, cfg.D
    prm = synth.torch_params(cfg, 3, dev, bo_scale=0.05)
    prm["Wo"] *= 5.0
    opt = PPOOptimizer(D, H, B, T, cfg.head_sizes, precision="bf16")
    opt.load_canonical(prm["Wx"], prm["Wh"], prm["b"], prm["Wo"], prm["bo"])
    p64 = {k: v.double().cpu().numpy() for k, v in prm.items()}
    seq = synth.torch_sequences(cfg, 5, dev)
    R = B * T // 256
    ro = synth.torch_rollouts(R, 256, 5, dev, p_done=0.01)
    valid = torch.zeros((T, B), dtype=torch.uint8, device=dev)
    for b in SAMPLE_SEQ:
        valid[:, b] = 1
    # host copies of the sampled sequences (inputs are synth draws, not CUDA-path outputs)
    sidx = list(SAMPLE_SEQ)
    hseq = dict(x=seq["x"][:, sidx].float().cpu().numpy(), h0=seq["h0"][sidx].cpu().numpy(),
                c0=seq["c0"][sidx].cpu().numpy(), act=seq["act"][:, sidx].cpu().numpy(),
                head_on=seq["head_on"][:, sidx].cpu().numpy(),
                avail=seq["avail"][:, sidx].cpu().numpy(),
                valid=np.ones((T, len(sidx)), np.uint8))
    # oracle GAE for the streams holding the sampled sequences (sequence b = r*16 + k)
    gamma32 = float(np.float32(oracle.gamma_from_horizon(HYPER["horizon_s"], HYPER["T_step"])))
    lam32 = float(np.float32(HYPER["lam"]))
    streams = sorted(set(SAMPLE_STREAMS) | {b // 16 for b in SAMPLE_SEQ})
    r_np = ro["rew"][streams].cpu().numpy()
    v_np = ro["val"][streams].cpu().numpy()
    d_np = ro["done"][streams].cpu().numpy()
    A_o, R_o = oracle.gae(r_np, v_np, d_np, gamma32, lam32)
    gae_ref = {r: (A_o[i], R_o[i]) for i, r in enumerate(streams)}
    adv_s = np.stack([[gae_ref[b // 16][0][(b % 16) * 16 + t] for b in SAMPLE_SEQ] for t in range(T)])
    ret_s = np.stack([[gae_ref[b // 16][1][(b % 16) * 16 + t] for b in SAMPLE_SEQ] for t in range(T)])
    # behaviour log-probs of the sampled rows from the oracle's own forward pass + noise
    cache = oracle.lstm_forward(p64["Wx"], p64["Wh"], p64["b"], hseq["x"], hseq["h0"], hseq["c0"])
    Y_s = oracle.heads_forward(cache["h"].reshape(T * len(sidx), H), p64["Wo"], p64["bo"])
    lp_s = oracle.ppo_loss(Y_s, hseq["act"], hseq["head_on"], hseq["avail"],
                           np.zeros(T * len(sidx)), adv_s, ret_s, None,
                           cfg.head_sizes)[3].reshape(T, len(sidx))
    noise = seq["logp_noise"][:, sidx].double().cpu().numpy()
    lp_old_s = (lp_s + noise).astype(np.float32)
    logp_old = torch.zeros((T, B), device=dev)
    logp_old[:, sidx] = torch.from_numpy(lp_old_s).to(dev)
    batch = dict(x=seq["x"], h0=seq["h0"], c0=seq["c0"], act=seq["act"], head_on=seq["head_on"],
                 avail=seq["avail"], valid=valid, logp_old=logp_old, rew=ro["rew"],
                 val=ro["val"], done=ro["done"])
    theta0 = opt.theta.clone()
    opt.step(batch)
    torch.cuda.synchronize()
    # oracle: loss/grads over the sampled sequences with the full-batch denominator
    Lref, gref, st, inter = loss_and_grads(p64, hseq, lp_old_s.astype(np.float64), adv_s, ret_s,
                                           cfg.head_sizes, HYPER["clip_eps"], HYPER["c_v"],
                                           HYPER["c_e"], denom=float(T * B))
    return dict(cfg=cfg, opt=opt, batch=batch, theta0=theta0, gae_ref=gae_ref, gref=gref, st=st,
                inter=inter, sidx=sidx, adv_s=adv_s, ret_s=ret_s, lp_old_s=lp_old_s)


def test_gae_sampled_streams(run):
    opt, T = run["opt"], run["cfg"].T
    adv = opt.adv.cpu().numpy()
    ret = opt.ret.cpu().numpy()
    for r, (A, R) in run["gae_ref"].items():
        got_a = np.array([adv[l % 16, r * 16 + l // 16] for l in range(256)])
        got_r = np.array([ret[l % 16, r * 16 + l // 16] for l in range(256)])
        ok, worst = elementwise_ok(got_a, A, 1e-5)
        assert ok, (r, worst)
        ok, worst = elementwise_ok(got_r, R, 1e-5)
        assert ok, (r, worst)


def test_forward_sampled_sequences(run):
    opt, T, B = run["opt"], run["cfg"].T, run["cfg"].B
    Y = opt.out.view(T, B, -1)[:, run["sidx"]].cpu().numpy().reshape(T * len(run["sidx"]), -1)
    e = normwise(Y, run["inter"]["Y"])
    assert e < 2e-2, e


def test_loss_rows_sampled(run):
    """dL/dy of the sampled rows from the oracle loss fed the GPU's own head outputs (the
    loss is row-local given y), with the full-batch denominator."""
    opt, T, B = run["opt"], run["cfg"].T, run["cfg"].B
    sidx = run["sidx"]
    Y = opt.out.view(T, B, -1)[:, sidx].cpu().numpy().reshape(T * len(sidx), -1)
    b = run["batch"]
    pick = lambda k: b[k][:, sidx].cpu().numpy().reshape(T * len(sidx), -1)
    _, dYref, _, lpref = oracle.ppo_loss(Y, pick("act"), pick("head_on"), pick("avail"),
                                         run["lp_old_s"].reshape(-1), run["adv_s"].reshape(-1),
                                         run["ret_s"].reshape(-1), None, run["cfg"].head_sizes,
                                         HYPER["clip_eps"], HYPER["c_v"], HYPER["c_e"],
                                         denom=float(T * B))
    d = opt.dout.view(T, B, -1)[:, sidx].float().cpu().numpy().reshape(T * len(sidx), -1)
    # one bf16 rounding of an fp32 result that meets the fp32 bar (1e-5 of |ref| + rms(ref),
    # elementwise_ok): entries 1e-6 of their row's largest (p ~ 1e-6, cek y + c1 cancelling)
    # carry fp32 errors that are small against the rms but not against themselves
    rms = np.sqrt(np.mean(dYref * dYref))
    bound = 2 ** -8 * np.abs(dYref) + 1e-5 * (np.abs(dYref) + rms)
    bad = np.argwhere(np.abs(d - dYref) > bound)
    rowmax = np.abs(dYref).max(axis=1)
    assert bad.size == 0, [(int(i), int(j), float(dYref[i, j]), float(d[i, j]), float(rowmax[i]))
                           for i, j in bad[:8]]
    lp = opt.logp.view(T, B)[:, sidx].cpu().numpy().reshape(-1)
    ok, worst = elementwise_ok(lp, lpref, 1e-5)
    assert ok, worst
    # every other row is masked: exactly zero gradient
    mask = torch.ones(B, dtype=torch.bool, device="cuda")
    mask[sidx] = False
    dout = opt.dout.view(T, B, -1)
    for t in range(T):  # one time slice at a time: no multi-GB temporary at B_max
        assert int(torch.count_nonzero(dout[t, mask])) == 0, t


def test_weight_gradients_masked_batch(run):
    g = {k: v.cpu().numpy() for k, v in run["opt"].unpack(run["opt"].grad).items()}
    for k in ("Wx", "Wh", "b", "Wo", "bo"):
        e = normwise(g[k], run["gref"][k])
        assert e < 2e-2, (k, e)


def test_adam_sampled_elements(run):
    opt = run["opt"]
    n = opt.theta.numel()
    idx = torch.from_numpy(np.random.default_rng(0).integers(0, n, 20000)).cuda()
    p0 = run["theta0"][idx].double().cpu().numpy()
    g = opt.grad[idx].double().cpu().numpy()
    z = np.zeros_like(p0)
    pr, mr, vr = oracle.adam_clip(p0, g, z, z, 1, HYPER["lr"], HYPER["beta1"], HYPER["beta2"],
                                  HYPER["adam_eps"], HYPER["clip_sigma"])
    got = opt.theta[idx].double().cpu().numpy()
    assert np.all(np.abs(got - pr) <= 1e-6 * (np.abs(p0) + np.abs(pr - p0)) + 1e-30)
    assert np.array_equal(opt.m[idx].double().cpu().numpy() != 0, g != 0)
