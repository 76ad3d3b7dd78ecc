"""End-to-end parity of one PPO optimizer step (a1-a10) on the GPU against the oracle.

Tolerances (north_star / DESIGN.md "Parity"): GAE and loss scalars 1e-5 relative; fp32
reference path: gradients and updates normwise 1e-4; bf16 tensor-core path: gradients and
outputs normwise 2e-2, updates checked where the gradient sign is resolved."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import HYPER, device_batch, elementwise_ok, load_params, make_case, normwise

pytestmark = pytest.mark.gpu

KEYS = ("Wx", "Wh", "b", "Wo", "bo")
# bf16 path: the share of entries whose gradient sign the GPU resolves (|g_ref| > 3|g - g_ref|);
# measured 0.984-1.000 over every tensor of the bf16 step tests (profiles/r02_gpu_tests_v1.txt)
BF16_FIRM_FLOOR = 0.95


def _run(case, cfg, precision):
    from paper_1912_06680_b200 import PPOOptimizer
    opt = PPOOptimizer(cfg.D, cfg.H, cfg.B, cfg.T, cfg.head_sizes, precision=precision)
    load_params(opt, case["params"])
    batch = device_batch(case, precision == "bf16")
    theta0 = opt.theta.clone()
    stats = opt.step(batch).cpu().numpy()
    torch.cuda.synchronize()
    return opt, batch, theta0, stats


def _check_step(case, cfg, precision, tol_fwd, tol_grad, stat_floor=1e-3):
    opt, batch, theta0, stats = _run(case, cfg, precision)
    T, B, A = cfg.T, cfg.B, cfg.A
    # a1: GAE in minibatch layout
    ok, worst = elementwise_ok(opt.adv.cpu().numpy(), case["adv"], 1e-5)
    assert ok, worst
    ok, worst = elementwise_ok(opt.ret.cpu().numpy(), case["ret"], 1e-5)
    assert ok, worst
    # a2-a4: head outputs
    Y = opt.out.cpu().numpy()
    e = normwise(Y, case["inter"]["Y"])
    assert e < tol_fwd, ("out", e)
    # a5: loss statistics
    st = case["stats"]
    tol_s = 1e-5 if precision == "fp32" else 2e-2
    for i, k in enumerate(("loss", "pg", "vf", "ent")):
        assert abs(stats[i] - st[k]) <= tol_s * (abs(st[k]) + stat_floor), (k, stats[i], st[k])
    assert stats[6] == st["n_valid"] and int(stats[7]) == 0
    # a6-a8: gradients (canonical layout)
    g = {k: v.cpu().numpy() for k, v in opt.unpack(opt.grad).items()}
    for k in KEYS:
        e = normwise(g[k], case["grads"][k])
        assert e < tol_grad, (k, e)
    # a10: Adam update against the oracle applied to the oracle gradient
    new = {k: v.cpu().numpy().astype(np.float64) for k, v in opt.unpack(opt.theta).items()}
    old = {k: v.cpu().numpy().astype(np.float64) for k, v in opt.unpack(theta0).items()}
    for k in KEYS:
        zeros = np.zeros_like(old[k])
        ref, _, _ = oracle.adam_clip(old[k], case["grads"][k], zeros, zeros, 1, HYPER["lr"],
                                     HYPER["beta1"], HYPER["beta2"], HYPER["adam_eps"],
                                     HYPER["clip_sigma"])
        d_ref = ref - old[k]
        d_got = new[k] - old[k]
        if precision == "fp32":
            # Adam's first step is ~ -alpha/2 sign(g) (eps/sqrt(v) matters only for tiny |g|):
            # compare where the gradient itself agrees to 1e-4 relative (>= 90% of entries)
            # theta is fp32: the reference update is the fp32 rounding of old + d_ref, since
            # ulp(theta) (~4e-9 at |theta| ~ 0.05) is ~1e-4 of the first update (~1e-5)
            d_ref = (old[k] + d_ref).astype(np.float32).astype(np.float64) - old[k]
            gerr = np.abs(g[k] - case["grads"][k])
            firm = np.abs(case["grads"][k]) > 1e4 * gerr
            assert firm.mean() > 0.9, (k, firm.mean())
            e = normwise(d_got[firm], d_ref[firm])
            assert e < 1e-4, (k, e, firm.mean())
        else:
            # first Adam step ~ -alpha/2 sign(g): compare where the sign is resolved
            gerr = np.abs(g[k] - case["grads"][k])
            firm = np.abs(case["grads"][k]) > 3 * gerr + 1e-6
            assert firm.mean() > BF16_FIRM_FLOOR, (k, firm.mean())
            e = normwise(d_got[firm], d_ref[firm])
            assert e < 2e-2, (k, e, firm.mean())
    return opt


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_tiny_step_fp32(seed):
    cfg = synth.TINY
    case = make_case(cfg, seed, pad_frac=0.25, wo_scale=20.0)
    _check_step(case, cfg, "fp32", 1e-4, 1e-4)


@pytest.mark.parametrize("seed", [0, 1])
def test_tiny_step_bf16(seed):
    cfg = synth.TINY
    case = make_case(cfg, seed, pad_frac=0.25, wo_scale=20.0)
    _check_step(case, cfg, "bf16", 2e-2, 2e-2)


def test_ragged_batch_bf16():
    """B not a multiple of the 128-row tile; D != H; several tiles in every GEMM."""
    cfg = synth.Config(H=256, D=192, B=176)
    case = make_case(cfg, 4, pad_frac=0.1, wo_scale=10.0)
    _check_step(case, cfg, "bf16", 2e-2, 2e-2)


def test_ragged_batch_fp32():
    cfg = synth.Config(H=256, D=192, B=176)
    case = make_case(cfg, 4, pad_frac=0.1, wo_scale=10.0)
    _check_step(case, cfg, "fp32", 1e-4, 1e-4)


def test_full_width_bf16():
    """The paper's LSTM-4096 with D = 4032 (DESIGN Q1) on B = 48 sequences."""
    cfg = synth.Config(H=4096, D=4032, B=48)
    case = make_case(cfg, 7, pad_frac=0.1, wo_scale=5.0)
    _check_step(case, cfg, "bf16", 2e-2, 2e-2)


def test_split_k_backward_bf16():
    """Small minibatch (fewer backward tiles per step than CTA pairs): the backward step GEMM
    runs split-K into fp32 partials and the cell backward as a separate coalesced kernel
    (tc_path.cu bwd_split): H = 2048 (K = 4H + A = 139 k-blocks -> 2 splits), 2 x 8 tiles."""
    cfg = synth.Config(H=2048, D=512, B=288)
    # wo_scale 4: with 8 the bf16 forward alone leaves 5% of W_h's entries sign-unresolved
    # for the split and the fused backward alike (profiles/r02_split_check.txt)
    case = make_case(cfg, 9, pad_frac=0.1, wo_scale=4.0)
    # pg = -mean(min(rho A, clip(rho) A)) is a cancelling mean (2.4e-3 here from terms of
    # order |A| ~ 1): the bf16 forward (computed before and independently of the backward
    # under test) moves it by 8.5e-5, so its absolute floor is 5e-3 x 2e-2 = 1e-4
    _check_step(case, cfg, "bf16", 2e-2, 2e-2, stat_floor=5e-3)


def test_determinism_bf16():
    cfg = synth.TINY
    case = make_case(cfg, 3)
    o1 = _run(case, cfg, "bf16")[0]
    o2 = _run(case, cfg, "bf16")[0]
    assert torch.equal(o1.grad, o2.grad) and torch.equal(o1.theta, o2.theta)


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_dp_equivalence_shards(precision):
    """the average of N per-GPU gradients (each with its local denominator, Q9) equals
    the gradient of the concatenated batch.  The N ranks are emulated serially on one GPU
    (nothing waits on another launch); the average is the test's own reference arithmetic."""
    from paper_1912_06680_b200 import PPOOptimizer
    cfg = synth.Config(H=128, D=256, B=64)
    case = make_case(cfg, 11, pad_frac=0.2, wo_scale=20.0)
    full = device_batch(case, precision == "bf16")
    ref = PPOOptimizer(cfg.D, cfg.H, cfg.B, cfg.T, cfg.head_sizes, precision=precision)
    load_params(ref, case["params"])
    ref.step(full)
    N = 4
    Bs = cfg.B // N
    Rs = case["ro"]["r"].shape[0] // N
    acc = torch.zeros_like(ref.grad)
    for n in range(N):
        sl, rs = slice(n * Bs, (n + 1) * Bs), slice(n * Rs, (n + 1) * Rs)
        shard = {k: (v[:, sl] if k in ("x", "act", "head_on", "avail", "valid", "logp_old")
                     else v[sl] if k in ("h0", "c0") else v[rs]).contiguous()
                 for k, v in full.items()}
        o = PPOOptimizer(cfg.D, cfg.H, Bs, cfg.T, cfg.head_sizes, precision=precision)
        load_params(o, case["params"])
        o.step(shard)
        acc += o.grad
    acc /= N
    torch.cuda.synchronize()
    e = (torch.linalg.vector_norm(acc - ref.grad) / torch.linalg.vector_norm(ref.grad)).item()
    assert e < 1e-5, e


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_zero_copy_x_matches_packed(precision):
    """x placed in the workspace by ppo_copy_x (from pinned host and from device memory) gives
    the same forward outputs, bit for bit, as the packed path; ragged B, two workspaces."""
    from paper_1912_06680_b200 import PPOOptimizer, _lib as L
    cfg = synth.Config(H=256, D=192, B=176, T=16)
    case = make_case(cfg, 5, pad_frac=0.2)
    opt = PPOOptimizer(cfg.D, cfg.H, cfg.B, cfg.T, cfg.head_sizes, precision=precision, n_ws=2)
    load_params(opt, case["params"])
    batch = device_batch(case, precision == "bf16")
    opt.forward(batch)
    ref = opt.out.clone()
    xh = batch["x"].cpu().pin_memory()
    for ws, src in ((1, xh), (0, batch["x"])):
        opt.out.zero_()
        opt.put_x(src, ws=ws)
        opt.select_ws(ws)
        opt.forward(dict(batch, x=None))
        torch.cuda.synchronize()
        assert torch.equal(opt.out, ref), ws
    # streamed: x slice by slice on a side stream, the forward waits per time step
    side = torch.cuda.Stream()
    evs = [torch.cuda.Event() for _ in range(cfg.T)]
    opt.out.zero_()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for t in range(cfg.T):
            L.ppo_copy_x_slice(opt.dims, cfg.B, t, xh[t], opt.ws_list[1], side)
            evs[t].record(side)
    opt.select_ws(1)
    opt.forward_streamed(dict(batch, x=None), evs)
    torch.cuda.synchronize()
    assert torch.equal(opt.out, ref)
    p, ld = L.lstm_ws_x(opt.dims, cfg.B, opt.ws_list[1])
    assert p == opt.ws_list[1].data_ptr() and ld == cfg.D + cfg.H + 64
    with pytest.raises(RuntimeError):
        opt.forward(dict(batch, x=None, c0=None))


def test_lstm2048_full_width_bf16():
    """NEXT-4: the LSTM-2048 variant (the hidden size before the 4096 surgery)
    with the paper's D = 4032 (DESIGN Q1)."""
    cfg = synth.Config(H=2048, D=4032, B=48)
    case = make_case(cfg, 9, pad_frac=0.1, wo_scale=5.0)
    _check_step(case, cfg, "bf16", 2e-2, 2e-2)


def test_lstm2048_fp32():
    cfg = synth.Config(H=2048, D=4032, B=16)
    case = make_case(cfg, 10, pad_frac=0.1, wo_scale=5.0)
    _check_step(case, cfg, "fp32", 1e-4, 1e-4)


@pytest.mark.parametrize("precision,H,D,B,tol", [("fp32", 256, 192, 176, 1e-4),
                                                 ("bf16", 256, 192, 176, 2e-2),
                                                 ("bf16", 4096, 4032, 48, 2e-2)])
def test_input_grad(precision, H, D, B, tol):
    """NEXT-4: dL/dx for the observation-processing network (lstm_input_grad) against the
    oracle's dz W_x (oracle.lstm_input_grad, pinned to autograd)."""
    from paper_1912_06680_b200 import PPOOptimizer
    cfg = synth.Config(H=H, D=D, B=B)
    case = make_case(cfg, 6, pad_frac=0.1, wo_scale=10.0)
    opt = PPOOptimizer(cfg.D, cfg.H, cfg.B, cfg.T, cfg.head_sizes, precision=precision)
    load_params(opt, case["params"])
    batch = device_batch(case, precision == "bf16")
    opt.gae(batch)
    opt.forward(batch)
    opt.loss(batch)
    opt.backward()
    dx = torch.full((cfg.T, cfg.B, cfg.D), float("nan"), device="cuda")
    opt.input_grad(dx)
    torch.cuda.synchronize()
    ref = oracle.lstm_input_grad(case["params"]["Wx"], case["inter"]["dz"])
    e = normwise(dx.cpu().numpy(), ref)
    assert e < tol, e


@pytest.mark.parametrize("precision,T,B", [("fp32", 4, 64), ("bf16", 4, 64), ("bf16", 1, 256),
                                           ("fp32", 1, 256)])
def test_other_unroll_lengths(precision, T, B):
    """TBPTT over T != 16 (the paper's 16, is a parameter): T = 4, and T = 1 where the
    backward has only the last step (no recurrent term)."""
    cfg = synth.Config(H=128, D=128, B=B, T=T)
    case = make_case(cfg, 12, pad_frac=0.2, wo_scale=10.0)
    tol = 1e-4 if precision == "fp32" else 2e-2
    _check_step(case, cfg, precision, tol, tol)


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_checkpoint_resume(tmp_path, precision):
    """Save after two steps, resume into a fresh optimizer: the third step is bit-identical
    to the uninterrupted run (params, Adam moments and t round-trip through the canonical
    layout)."""
    from paper_1912_06680_b200 import PPOOptimizer
    cfg = synth.Config(H=128, D=256, B=32)
    case = make_case(cfg, 21, pad_frac=0.1, wo_scale=10.0)
    batch = device_batch(case, precision == "bf16")
    a = PPOOptimizer(cfg.D, cfg.H, cfg.B, cfg.T, cfg.head_sizes, precision=precision)
    load_params(a, case["params"])
    a.step(batch)
    a.step(batch)
    path = str(tmp_path / "ckpt.pt")
    a.save(path)
    b = PPOOptimizer(cfg.D, cfg.H, cfg.B, cfg.T, cfg.head_sizes, precision=precision)
    b.load(path)
    assert b.t == 2
    assert torch.equal(a.theta, b.theta) and torch.equal(a.m, b.m) and torch.equal(a.v, b.v)
    a.step(batch)
    b.step(batch)
    torch.cuda.synchronize()
    assert torch.equal(a.theta, b.theta) and torch.equal(a.grad, b.grad)
