"""The fused a9+a10 exchange (ppo_dp_adam_step) on one GPU: with a world-1 communicator the
rank owns the whole of theta, so two steps through the fused kernel must leave theta, m, v
and the bf16 shadow bit-identical to the allreduce + adam_step path (same arithmetic, same
order: the sum over one rank is the gradient itself, the scale 1/1 is exact).  The N > 1
parity against one GPU on the whole batch is tools/dist_parity.py --dp fused
(profiles/r01_dp_fused_parity.txt); the host-side checks are in test_abi.py."""
import pytest
import torch

import synth
from gpu_util import device_batch, load_params, make_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_fused_exchange_world1_bitwise(precision):
    from paper_1912_06680_b200 import PPOOptimizer, _lib as L
    cfg = synth.Config(H=128, D=256, B=32)
    case = make_case(cfg, 11, pad_frac=0.1, wo_scale=10.0)
    comm = L.comm_init(L.comm_unique_id(), 0, 1)
    try:
        opts = []
        for dp, c in (("fused", comm), ("allreduce", None)):
            opt = PPOOptimizer(cfg.D, cfg.H, cfg.B, cfg.T, cfg.head_sizes, precision=precision,
                               comm=c, dp=dp)
            assert opt.dp == dp
            load_params(opt, case["params"])
            batch = device_batch(case, precision == "bf16")
            for _ in range(2):
                opt.step(batch)
            opt.gather_sharded()
            torch.cuda.synchronize()
            opts.append(opt)
        f, r = opts
        assert L.dp_shard(f.layout.n_total, 1) >= f.layout.n_total
        for k in ("theta", "m", "v", "grad"):
            assert torch.equal(getattr(f, k), getattr(r, k)), k
        if precision == "bf16":
            assert torch.equal(f.shadow, r.shadow)
        assert not torch.equal(f.theta, f.theta * 0)          # something was updated
    finally:
        L.comm_destroy(comm)
