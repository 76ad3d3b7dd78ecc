"""NEXT-4 aux heads on the GPU: ppo_aux_labels and a full backward with aux heads against the
oracle (oracle/aux.py through oracle.step.loss_and_grads(aux=...)).

Tolerances: labels 1e-5 relative (fp32 recursion vs fp64, gamma2
fp32-rounded on both sides); loss statistics 1e-5 (fp32 path) / 2e-2 (bf16 path); head
outputs and gradients normwise 1e-4 (fp32) / 2e-2 (bf16).  win_trunk = 0.5 makes the win
head's route into the LSTM visible in dW_x; win_trunk = 0 makes every aux head stop_gradient.
"""
import numpy as np
import pytest
import torch

import synth
from gpu_util import AUX_HYPER, aux_case, dev, device_batch, elementwise_ok, load_params, \
    make_case, normwise

pytestmark = pytest.mark.gpu
KEYS = ("Wx", "Wh", "b", "Wo", "bo")
AUX = synth.AUX_SIZES


@pytest.mark.parametrize("seq_T", [0, 16])
def test_aux_labels_kernel(seq_T):
    from paper_1912_06680_b200 import _lib as L
    cfg = synth.Config(H=128, D=128, B=48, aux=AUX)
    R, Lseg = 3, 256
    ax, g2, lab, aux = aux_case(cfg, R, Lseg, 4, AUX_HYPER)
    dims = L.make_dims(cfg.D, cfg.H, cfg.T, cfg.head_sizes, L.PPO_PREC_BF16, AUX, 0.01)
    out = torch.full((R * Lseg * sum(AUX),), float("nan"), device="cuda")
    L.ppo_aux_labels(dims, dev(ax["last"]), dev(ax["outcome"]), dev(ax["rank"]),
                     dev(ax["events"]), dev(ax["boot"]), g2, out, seq_T=seq_T)
    torch.cuda.synchronize()
    ref = lab if seq_T == 0 else aux["labels"]
    got = out.cpu().numpy().reshape(ref.shape)
    assert np.allclose(got, ref, rtol=1e-5, atol=1e-7), np.abs(got - ref).max()
    assert ax["last"].any() and ax["events"].any()


def _grads(cfg, precision, trunk, seed, pad=0.1, wo=10.0):
    from paper_1912_06680_b200 import PPOOptimizer
    hyper = dict(AUX_HYPER, aux_win_trunk=trunk)
    case = make_case(cfg, seed, pad_frac=pad, wo_scale=wo, aux_hyper=hyper)
    opt = PPOOptimizer(cfg.D, cfg.H, cfg.B, cfg.T, cfg.head_sizes, precision=precision,
                       aux=cfg.aux, hyper=hyper)
    load_params(opt, case["params"])
    batch = device_batch(case, precision == "bf16")
    opt.gae(batch)
    opt.forward(batch)
    opt.loss(batch)
    opt.backward()
    torch.cuda.synchronize()
    return opt, case


@pytest.mark.parametrize("precision,trunk", [("fp32", 0.5), ("fp32", 0.0), ("bf16", 0.5),
                                             ("bf16", 0.0)])
def test_step_with_aux_heads(precision, trunk):
    cfg = synth.Config(H=128, D=256, B=32, aux=AUX)
    opt, case = _grads(cfg, precision, trunk, 3)
    tol = 1e-4 if precision == "fp32" else 2e-2
    st = opt.stats.cpu().numpy()
    ref = case["stats"]
    tol_s = 1e-5 if precision == "fp32" else 2e-2
    assert abs(st[0] - ref["loss"]) <= tol_s * (abs(ref["loss"]) + 1e-3), (st[0], ref["loss"])
    assert abs(st[8] - ref["aux"]) <= tol_s * (abs(ref["aux"]) + 1e-3), (st[8], ref["aux"])
    assert int(st[7]) == 0
    assert normwise(opt.out.cpu().numpy(), case["inter"]["Y"]) < tol
    g = {k: v.cpu().numpy() for k, v in opt.unpack(opt.grad).items()}
    for k in KEYS:
        e = normwise(g[k], case["grads"][k])
        assert e < tol, (k, e)
    # the aux rows of W_o (their own weights) separately: full gradient of their losses
    A0 = sum(cfg.head_sizes) + 1
    e = normwise(g["Wo"][A0:], case["grads"]["Wo"][A0:])
    assert e < tol, ("Wo aux rows", e)


def test_trunk_route_is_visible():
    """Sensitivity: with win_trunk 0.5 vs 0 the LSTM gradients differ by about as much as the
    oracle says, so the routing above is actually exercised."""
    cfg = synth.Config(H=128, D=256, B=32, aux=AUX)
    o1, c1 = _grads(cfg, "fp32", 0.5, 3)
    g1 = o1.unpack(o1.grad)["Wx"].cpu().numpy()
    o0, c0 = _grads(cfg, "fp32", 0.0, 3)
    g0 = o0.unpack(o0.grad)["Wx"].cpu().numpy()
    d_ref = c1["grads"]["Wx"] - c0["grads"]["Wx"]
    assert np.linalg.norm(d_ref) > 1e-3 * np.linalg.norm(c1["grads"]["Wx"])
    assert normwise(g1 - g0, d_ref) < 1e-3


def test_full_width_with_aux_bf16():
    cfg = synth.Config(H=4096, D=4032, B=48, aux=AUX)
    opt, case = _grads(cfg, "bf16", 0.01, 5, wo=5.0)
    assert normwise(opt.out.cpu().numpy(), case["inter"]["Y"]) < 2e-2
    g = {k: v.cpu().numpy() for k, v in opt.unpack(opt.grad).items()}
    for k in KEYS:
        assert normwise(g[k], case["grads"][k]) < 2e-2, k
