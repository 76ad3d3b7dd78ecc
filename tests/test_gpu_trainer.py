"""NEXT-1 on the GPU: experience buffer ingest (GAE at ingest), the minibatch sampler, the
gather into the forward workspace, and gradient steps drawn from the buffer vs the oracle."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import HYPER, dev, elementwise_ok, normwise
from oracle.step import loss_and_grads

pytestmark = pytest.mark.gpu
KEYS = ("Wx", "Wh", "b", "Wo", "bo")


def _segments(cfg, nseg, seed, bf16):
    """nseg rollout segments of 256 steps = 16*nseg sequences (host numpy + device tensors)."""
    c = synth.Config(H=cfg.H, D=cfg.D, B=16 * nseg, T=cfg.T)
    s = synth.make_sequences(c, seed, pad_frac=0.2)
    ro = synth.make_rollouts(nseg, 256, seed, p_done=0.01)
    # sequence-major host copies [n][T][.]
    host = dict(x=np.swapaxes(s["x"], 0, 1), h0=s["h0"], c0=s["c0"],
                act=np.swapaxes(s["act"], 0, 1), head_on=np.swapaxes(s["head_on"], 0, 1),
                avail=np.swapaxes(s["avail"], 0, 1), valid=np.swapaxes(s["valid"], 0, 1),
                logp_old=np.swapaxes(s["logp_noise"], 0, 1) - 3.0)
    d = {k: dev(np.ascontiguousarray(v)) for k, v in host.items()}
    if bf16:
        d["x"] = d["x"].bfloat16()
    d.update(rew=dev(ro["r"]), val=dev(ro["V"]), done=dev(ro["done"]))
    return host, ro, d


def _trainer(cfg, cap, precision, seed=0):
    from paper_1912_06680_b200 import PPOOptimizer
    from paper_1912_06680_b200.trainer import ExperienceBuffer, PPOTrainer
    opt = PPOOptimizer(cfg.D, cfg.H, cfg.B, cfg.T, cfg.head_sizes, precision=precision)
    prm = synth.make_params(cfg, 3, bo_scale=0.05)
    prm["Wo"] = prm["Wo"] * 20.0
    opt.load_canonical(*(dev(prm[k]) for k in KEYS))
    buf = ExperienceBuffer(cap, cfg.D, cfg.H, cfg.T, cfg.head_sizes, bf16=precision == "bf16")
    return opt, buf, PPOTrainer(opt, buf, seed=seed), prm


def _gamma():
    return (float(np.float32(oracle.gamma_from_horizon(HYPER["horizon_s"], HYPER["T_step"]))),
            float(np.float32(HYPER["lam"])))


def test_sampler_bit_exact():
    from paper_1912_06680_b200 import _lib as L
    for cap, B, seed, step in ((97, 5000, 5, 3), (1 << 20, 4096, 123, 77), (64, 1, 0, 0)):
        idx = torch.empty(B, dtype=torch.int32, device="cuda")
        L.ppo_sample_indices(cap, B, seed, step, idx)
        torch.cuda.synchronize()
        assert np.array_equal(idx.cpu().numpy(), oracle.buffer.sample_indices(cap, B, seed, step))


def test_ingest_gae_and_gather():
    from paper_1912_06680_b200 import _lib as L
    cfg = synth.Config(H=128, D=256, B=48)
    opt, buf, tr, _ = _trainer(cfg, cap=96, precision="bf16")
    g, lam = _gamma()
    host, ro, d = _segments(cfg, 6, 1, True)
    buf.push_segments(d, g, lam)
    A, R = oracle.gae(ro["r"], ro["V"], ro["done"], g, lam)
    ok, worst = elementwise_ok(buf.t["adv"].cpu().numpy().reshape(6, 256), A, 1e-5)
    assert ok, worst
    ok, worst = elementwise_ok(buf.t["ret"].cpu().numpy().reshape(6, 256), R, 1e-5)
    assert ok, worst
    # gather -> forward(x=None) == forward on the same minibatch passed explicitly (bitwise)
    tr.step()  # advances the sampler; uses step 0
    torch.cuda.synchronize()
    idx = oracle.buffer.sample_indices(96, cfg.B, 0, 0)
    assert np.array_equal(tr.idx.cpu().numpy(), idx)
    gath = oracle.buffer.gather({k: buf.t[k].cpu().numpy() for k in
                                 ("act", "head_on", "avail", "logp_old", "adv", "ret", "valid")}, idx)
    for k in ("act", "head_on", "avail", "logp_old", "valid"):
        assert np.array_equal(tr.mb[k].cpu().numpy(), gath[k]), k
    assert np.array_equal(opt.adv.cpu().numpy(), gath["adv"])
    assert np.array_equal(opt.ret.cpu().numpy(), gath["ret"])
    out_gather = opt.out.clone()
    xg = buf.t["x"][torch.from_numpy(idx).cuda()].transpose(0, 1).contiguous()
    h0 = buf.t["h0"][torch.from_numpy(idx).cuda()].contiguous()
    c0 = buf.t["c0"][torch.from_numpy(idx).cuda()].contiguous()
    # the step above updated theta; recompute the gathered forward with the new weights too
    L.ppo_gather(opt.dims, buf.view, tr.idx, cfg.B, opt.ws, tr.mb["act"], tr.mb["head_on"],
                 tr.mb["avail"], tr.mb["logp_old"], opt.adv, opt.ret, tr.mb["valid"])
    opt.forward(dict(x=None, h0=None, c0=None))
    out_g2 = opt.out.clone()
    opt.forward(dict(x=xg, h0=h0, c0=c0))
    torch.cuda.synchronize()
    assert torch.equal(out_g2, opt.out)
    assert out_gather.abs().sum() > 0


def test_steps_from_buffer_vs_oracle_fp32():
    """Two gradient steps drawn from the buffer (fp32 reference path) against the oracle
    drawing the same minibatches with its own sampler and gather."""
    cfg = synth.Config(H=128, D=256, B=32)
    opt, buf, tr, prm = _trainer(cfg, cap=64, precision="fp32", seed=9)
    g, lam = _gamma()
    host, ro, d = _segments(cfg, 4, 2, False)
    buf.push_segments(d, g, lam)
    A, R = oracle.gae(ro["r"], ro["V"], ro["done"], g, lam)
    hbuf = dict(host, adv=A.reshape(64, 16), ret=R.reshape(64, 16))
    p = {k: v.astype(np.float64) for k, v in prm.items()}
    state = {k: (np.zeros_like(v), np.zeros_like(v)) for k, v in p.items()}
    for step in range(2):
        stats = tr.step().cpu().numpy()
        torch.cuda.synchronize()
        idx = oracle.buffer.sample_indices(64, cfg.B, 9, step)
        mb = oracle.buffer.gather(hbuf, idx)
        seq = {k: mb[k] for k in ("x", "h0", "c0", "act", "head_on", "avail", "valid")}
        Lref, gref, st, _ = loss_and_grads(p, seq, mb["logp_old"], mb["adv"], mb["ret"],
                                           cfg.head_sizes, HYPER["clip_eps"], HYPER["c_v"], HYPER["c_e"])
        assert abs(stats[0] - st["loss"]) <= 1e-5 * (abs(st["loss"]) + 1e-3), (step, stats[0], st["loss"])
        gg = {k: v.cpu().numpy() for k, v in opt.unpack(opt.grad).items()}
        for k in KEYS:
            assert normwise(gg[k], gref[k]) < 1e-4, (step, k, normwise(gg[k], gref[k]))
        # the oracle applies Adam to its own gradient for the next step
        for k in KEYS:
            m, v = state[k]
            p[k], m, v = oracle.adam_clip(p[k], gref[k], m, v, step + 1, HYPER["lr"],
                                          HYPER["beta1"], HYPER["beta2"], HYPER["adam_eps"],
                                          HYPER["clip_sigma"])
            state[k] = (m, v)


def test_iteration_publishes_version():
    cfg = synth.Config(H=128, D=256, B=32)
    opt, buf, tr, _ = _trainer(cfg, cap=64, precision="bf16")
    tr.steps_per_iteration = 3
    g, lam = _gamma()
    _, _, d = _segments(cfg, 4, 3, True)
    buf.push_segments(d, g, lam)
    before = tr.published.clone()
    v = tr.iteration()
    torch.cuda.synchronize()
    assert v == 1 and tr.global_step == 3
    assert torch.equal(tr.published, opt.shadow) and not torch.equal(before, tr.published)
    assert abs(tr.sample_reuse - 3 * 32 / 64) < 1e-12
