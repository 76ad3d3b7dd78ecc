"""The whole optimizer step (a1-a10) captured in one CUDA graph and the
device step counter of Adam that makes it replayable (adam_step_ctr).

* Graph replays equal eager steps bit for bit: an optimizer that runs 1 eager step, captures
  the step and replays it 3 times ends with the same theta, bf16 shadow, m, v, gradient and
  loss statistics as one that runs 4 eager steps (both with the device step counter), and its
  step count reads 4 -- for the multi-step launches (tiny, ragged) and the small-B split-K
  backward (H = 2048, B = 288: split GEMM + cell kernel per step).
* The device alpha_t equals the host one: adam_step_ctr and adam_step give the same bits for
  t = 1 ... 300 (alpha_t = lr sqrt(1 - b2^t) / (1 - b1^t) in double, rounded once to fp32 on
  either side, ppo5.h), so a graph-replayed run also equals a host-counter run.
* The step parity against the oracle (test_gpu_step.py) therefore carries over to replays.
"""
import numpy as np
import pytest
import torch

import synth
from gpu_util import dev, device_batch, load_params, make_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_1912_06680_b200 import _lib
    return _lib


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("cfg", [synth.TINY, synth.Config(H=256, D=192, B=176),
                                 synth.Config(H=2048, D=512, B=288)],
                         ids=["tiny", "ragged", "splitk"])
def test_graph_replay_equals_eager(L, precision, cfg):
    from paper_1912_06680_b200 import PPOOptimizer
    case = make_case(cfg, 8, pad_frac=0.2, wo_scale=10.0)
    opts = []
    for mode in ("eager", "graph"):
        opt = PPOOptimizer(cfg.D, cfg.H, cfg.B, cfg.T, cfg.head_sizes, precision=precision)
        load_params(opt, case["params"])
        batch = device_batch(case, precision == "bf16")
        opt.use_device_t()
        opt.step(batch)                      # eager step 1 (sets up kernels outside capture)
        if mode == "eager":
            for _ in range(3):
                opt.step(batch)
        else:
            g = opt.capture(batch)
            for _ in range(3):
                g.replay()
        torch.cuda.synchronize()
        opts.append(opt)
    e, gr = opts
    assert gr.sync_t() == 4 and e.sync_t() == 4
    for k in ("theta", "m", "v", "grad", "adv", "ret", "out", "dout"):
        assert torch.equal(getattr(e, k), getattr(gr, k)), k
    if precision == "bf16":
        assert torch.equal(e.shadow, gr.shadow)
    assert torch.equal(e.stats[:L.PPO_STATS], gr.stats[:L.PPO_STATS])
    assert int(gr.stats[7].item()) == 0
    assert not torch.equal(gr.theta, opts[0].theta * 0)


def test_device_alpha_equals_host_alpha(L):
    """adam_step_ctr (alpha_t on the device) == adam_step (alpha_t on the host) bit for bit
    over 300 consecutive steps, with the clip active early and the bf16 shadow."""
    n = 4099
    rng = np.random.default_rng(3)
    p0 = rng.standard_normal(n).astype(np.float32)
    P1, P2 = dev(p0), dev(p0)
    M1, M2 = (torch.zeros(n, device="cuda") for _ in range(2))
    V1, V2 = (torch.zeros(n, device="cuda") for _ in range(2))
    S1, S2 = (torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(2))
    ctr = torch.zeros(2, dtype=torch.int64, device="cuda")
    for t in range(1, 301):
        g = dev((rng.standard_normal(n) * np.exp(rng.uniform(-6, 2, n))).astype(np.float32))
        L.adam_step(P1, S1, g, M1, V1, t, 5e-5, 0.9, 0.999, 1e-8, 5.0)
        L.adam_step_ctr(P2, S2, g, M2, V2, ctr, 5e-5, 0.9, 0.999, 1e-8, 5.0)
    torch.cuda.synchronize()
    assert int(ctr[0].item()) == 300
    for a, b in ((P1, P2), (M1, M2), (V1, V2), (S1, S2)):
        assert torch.equal(a, b)


def test_capture_rejects_fused_exchange(L):
    from paper_1912_06680_b200 import PPOOptimizer
    cfg = synth.TINY
    comm = L.comm_init(L.comm_unique_id(), 0, 1)
    try:
        opt = PPOOptimizer(cfg.D, cfg.H, cfg.B, cfg.T, cfg.head_sizes, comm=comm, dp="fused")
        with pytest.raises(ValueError):
            opt.capture({})
    finally:
        L.comm_destroy(comm)
