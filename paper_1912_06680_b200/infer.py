"""NEXT-3: the forward-pass inference step -- thin wrapper over ppo_infer_step.

PolicyServer holds the bf16 weights it serves (a published parameter version), the
per-hero recurrent state (h, c) of a batch of B ~ 60 heroes and the workspace; each
call runs one LSTM step + heads + masked factorised sampling in libppo5's kernels.
"""
from __future__ import annotations

import torch

from . import _lib as L
from .step import HEAD_SIZES, _aligned_empty


class PolicyServer:
    def __init__(self, D: int, H: int, B: int, head_sizes=HEAD_SIZES, device="cuda",
                 head_table=None, seed: int = 0):
        self.D, self.H, self.B = D, H, B
        self.head_sizes = tuple(head_sizes)
        self.A = sum(self.head_sizes) + 1
        self.device = torch.device(device)
        self.dims = L.make_dims(D, H, 1, self.head_sizes, L.PPO_PREC_BF16)
        self.layout = L.param_layout(self.dims)
        dev = self.device
        # the served version, tiled for streaming (ppo_infer_pack_weights)
        self.wt = torch.zeros(L.infer_weights_bytes(self.dims) // 2, dtype=torch.bfloat16,
                              device=dev)
        self.h = torch.zeros(B, H, device=dev)
        self.c = torch.zeros(B, H, device=dev)
        nh, n0 = len(self.head_sizes), self.head_sizes[0]
        self.head_table = (torch.ones(n0, nh, dtype=torch.uint8, device=dev) if head_table is None
                           else head_table.to(dev, torch.uint8).contiguous())
        self.ws = _aligned_empty(L.infer_ws_bytes(self.dims, B), dev)
        self.act = torch.empty(B, nh, dtype=torch.int32, device=dev)
        self.head_on = torch.empty(B, nh, dtype=torch.uint8, device=dev)
        self.logp = torch.empty(B, device=dev)
        self.value = torch.empty(B, device=dev)
        self.out = torch.empty(B, self.A, device=dev)
        self.seed, self.t = seed, 0
        # the step counter lives on the device (ppo_infer_step_ctr): a captured CUDA graph of
        # steps draws fresh noise on every replay
        self.step_ctr = torch.zeros(1, dtype=torch.int64, device=dev)
        # the workspace's bf16 copy of h is current only after a step (reset() or an
        # external change of h invalidates it)
        self.state_current = False

    def load(self, weights: torch.Tensor, stream=None):
        """a published bf16 parameter vector (PPOOptimizer.shadow layout) -> tiled copy"""
        if weights.numel() != self.layout.n_total or weights.dtype != torch.bfloat16:
            raise ValueError("expected the bf16 parameter vector of ppo_param_layout")
        L.ppo_infer_pack_weights(self.dims, weights, self.wt, stream)

    def reset(self, h0=None, c0=None, step: int | None = None):
        self.h.copy_(h0) if h0 is not None else self.h.zero_()
        self.c.copy_(c0) if c0 is not None else self.c.zero_()
        if step is not None:
            self.step_ctr.fill_(step)
            self.t = step
        self.state_current = False

    def step(self, x: torch.Tensor, avail: torch.Tensor, want_out: bool = True, stream=None):
        """x [B][D] bf16, avail [B][n_primary] uint8 -> (act, head_on, logp, value); the
        recurrent state advances in place."""
        L.ppo_infer_step_ctr(self.dims, self.wt, x, self.h, self.c, avail, self.head_table,
                             self.seed, self.step_ctr, self.B, self.ws, self.act, self.head_on,
                             self.logp, self.value, self.out if want_out else None, stream,
                             flags=L.PPO_INFER_STATE_CURRENT if self.state_current else 0)
        self.state_current = True
        self.t += 1   # host mirror (eager calls only; graph replays advance step_ctr alone)
        return self.act, self.head_on, self.logp, self.value
