"""NEXT-2 on the GPU: reward pipeline fused into GAE vs oracle.reward + oracle.gae."""
import numpy as np
import pytest
import torch

import oracle
from oracle import reward
from gpu_util import dev, elementwise_ok

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G,L,tau,zs,seq_T", [(7, 256, 0.3, 1, 16), (5, 300, 0.8, 1, 0),
                                              (3, 64, 0.0, 0, 0), (64, 256, 1.0, 1, 16)])
def test_reward_gae_two_calls(G, L, tau, zs, seq_T):
    from paper_1912_06680_b200 import _lib as Lb
    rng = np.random.default_rng(G * 131 + L)
    gamma = float(np.float32(oracle.gamma_from_horizon(180.0)))
    lam = float(np.float32(0.95))
    cfg = Lb.ppo_reward_cfg(tau, 0.6, 600.0, float(np.float32(4.0 / 30.0)), zs)
    stats = torch.zeros(3, dtype=torch.float64, device="cuda")
    scratch = torch.empty(Lb.reward_gae_scratch_bytes(), dtype=torch.uint8, device="cuda")
    ostats = (0, 0.0, 0.0)
    for call in range(2):
        shaped = (0.3 * rng.standard_normal((G, 10, L))).astype(np.float32)
        win = ((rng.uniform(0, 1, (G, 10, L)) < 0.002) * 5.0).astype(np.float32)
        step0 = rng.integers(0, 20000, G).astype(np.int32)
        V = rng.standard_normal((G * 10, L + 1)).astype(np.float32)
        done = (rng.uniform(0, 1, (G, L)) < 0.01).astype(np.uint8)
        R = G * 10
        shape_out = (seq_T, R * L // seq_T) if seq_T else (R, L)
        adv = torch.empty(shape_out, device="cuda")
        ret = torch.empty(shape_out, device="cuda")
        rew = torch.empty((R, L), device="cuda")
        Lb.ppo_reward_gae(dev(shaped), dev(win), dev(step0), dev(V), dev(done), cfg, stats, gamma,
                          lam, adv, ret, scratch, seq_T=seq_T, rew_out=rew)
        torch.cuda.synchronize()
        # oracle: final rewards (fp32 step time as on the device), normalise, GAE per stream
        r = reward.shape_rewards(shaped, win, step0, tau, zero_sum=bool(zs))
        sigma, ostats = reward.running_std_update(ostats, r)
        rn = (r / sigma).reshape(R, L)
        d_streams = np.repeat(done, 10, axis=0)  # done is per game
        A, Rt = oracle.gae(rn, V, d_streams, gamma, lam)
        if seq_T:
            A = oracle.segments_to_sequences(A, seq_T)
            Rt = oracle.segments_to_sequences(Rt, seq_T)
        ok, worst = elementwise_ok(rew.cpu().numpy(), rn, 1e-5)
        assert ok, ("rew", call, worst)
        ok, worst = elementwise_ok(adv.cpu().numpy(), A, 1e-5)
        assert ok, ("adv", call, worst)
        ok, worst = elementwise_ok(ret.cpu().numpy(), Rt, 1e-5)
        assert ok, ("ret", call, worst)
        st = stats.cpu().numpy()
        assert st[0] == ostats[0]
        assert abs(st[1] - ostats[1]) <= 1e-6 * (abs(ostats[1]) + 1)
        assert abs(st[2] - ostats[2]) <= 1e-5 * ostats[2]
