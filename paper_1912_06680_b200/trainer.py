"""NEXT-1: the optimizer's experience buffer and the 32-step iteration.

ExperienceBuffer -- device-resident ring of `capacity` sequences; rollouts push 256-step
    segments whose GAE runs at ingest (ppo_gae, behaviour values).
PPOTrainer -- each gradient step samples a minibatch uniformly from the buffer
    (ppo_sample_indices), gathers it straight into the forward workspace (ppo_gather) and runs
    the step; every 32 steps it publishes a new parameter version (a bf16
    snapshot the forward-pass GPUs would pull).
All arithmetic runs in libppo5; torch only holds the memory.
"""
from __future__ import annotations

import torch

from . import _lib as L
from .step import PPOOptimizer

SEGMENT = 256  # steps per rollout segment


class ExperienceBuffer:
    def __init__(self, capacity: int, D: int, H: int, T: int, head_sizes, bf16: bool = True,
                 device="cuda"):
        if capacity % (SEGMENT // T):
            raise ValueError("capacity must hold whole segments")
        self.capacity, self.T = capacity, T
        self.seqs_per_segment = SEGMENT // T
        dev = torch.device(device)
        nh, n0 = len(head_sizes), head_sizes[0]
        self.t = dict(
            x=torch.zeros(capacity, T, D, dtype=torch.bfloat16 if bf16 else torch.float32, device=dev),
            h0=torch.zeros(capacity, H, device=dev), c0=torch.zeros(capacity, H, device=dev),
            act=torch.zeros(capacity, T, nh, dtype=torch.int32, device=dev),
            head_on=torch.zeros(capacity, T, nh, dtype=torch.uint8, device=dev),
            avail=torch.ones(capacity, T, n0, dtype=torch.uint8, device=dev),
            logp_old=torch.zeros(capacity, T, device=dev), adv=torch.zeros(capacity, T, device=dev),
            ret=torch.zeros(capacity, T, device=dev),
            valid=torch.zeros(capacity, T, dtype=torch.uint8, device=dev))
        self.pos = 0          # next slot (ring, whole segments)
        self.size = 0         # filled slots
        self.pushed = 0       # sequences ever pushed (for sample reuse)
        self.view = L.make_buffer(self.t, capacity)

    def push_segments(self, seg: dict, gamma: float, lam: float, stream=None):
        """seg: R segments as R*16 sequences -- x [R*16][T][D], h0/c0 [R*16][H] (recurrent state
        at each sequence start), act/head_on/avail/logp_old/valid [R*16][T][.], and the
        segments' rew [R][256], val [R][257] (bootstrap last), done [R][256]."""
        n = seg["x"].shape[0]
        R = seg["rew"].shape[0]
        assert n == R * self.seqs_per_segment and n <= self.capacity
        start = self.pos
        if start + n > self.capacity:
            start = 0
        sl = slice(start, start + n)
        for k in ("x", "h0", "c0", "act", "head_on", "avail", "logp_old"):
            self.t[k][sl].copy_(seg[k], non_blocking=True)
        self.t["valid"][sl].copy_(seg["valid"] if seg.get("valid") is not None else
                                  torch.ones_like(self.t["valid"][sl]), non_blocking=True)
        # GAE at ingest: the segment's 256 steps are contiguous in adv/ret of its 16 slots
        nb = L.gae_scratch_bytes(R, SEGMENT)
        scratch = torch.empty(nb, dtype=torch.uint8, device=self.t["adv"].device) if nb else None
        L.ppo_gae(seg["rew"], seg["val"], seg["done"], gamma, lam,
                  self.t["adv"][sl].view(R, SEGMENT), self.t["ret"][sl].view(R, SEGMENT),
                  seq_T=0, scratch=scratch, stream=stream)
        self.pos = (start + n) % self.capacity
        self.size = min(self.capacity, max(self.size, start + n))
        self.pushed += n


class PPOTrainer:
    def __init__(self, opt: PPOOptimizer, buffer: ExperienceBuffer, seed: int = 0,
                 steps_per_iteration: int = 32):
        self.opt, self.buf, self.seed = opt, buffer, seed
        self.steps_per_iteration = steps_per_iteration
        T, B, dev = opt.T, opt.B, opt.device
        nh, n0 = len(opt.head_sizes), opt.head_sizes[0]
        self.idx = torch.empty(B, dtype=torch.int32, device=dev)
        self.mb = dict(act=torch.empty(T, B, nh, dtype=torch.int32, device=dev),
                       head_on=torch.empty(T, B, nh, dtype=torch.uint8, device=dev),
                       avail=torch.empty(T, B, n0, dtype=torch.uint8, device=dev),
                       logp_old=torch.empty(T, B, device=dev),
                       valid=torch.empty(T, B, dtype=torch.uint8, device=dev))
        self.global_step = 0
        self.version = 0
        self.published = opt.weights.clone()   # the parameter version forward-pass GPUs pull
        self.consumed = 0

    def step(self, stream=None):
        """One gradient step on a minibatch sampled from the buffer; returns device stats."""
        opt, buf = self.opt, self.buf
        if buf.size < 1:
            raise RuntimeError("experience buffer is empty")
        L.ppo_sample_indices(buf.size, opt.B, self.seed, self.global_step, self.idx, stream)
        m = self.mb
        L.ppo_gather(opt.dims, buf.view, self.idx, opt.B, opt.ws, m["act"], m["head_on"],
                     m["avail"], m["logp_old"], opt.adv, opt.ret, m["valid"], stream)
        opt.forward(dict(x=None, h0=None, c0=None), stream)
        opt.loss(m, stream=stream)
        opt.backward(stream)
        opt.allreduce(stream)
        opt.apply(stream)
        self.global_step += 1
        self.consumed += opt.B
        return opt.stats[:L.PPO_STATS]

    def iteration(self, stream=None):
        """steps_per_iteration gradient steps, then publish a new version."""
        for _ in range(self.steps_per_iteration):
            self.step(stream)
        self.published.copy_(self.opt.weights, non_blocking=True)
        self.version += 1
        return self.version

    @property
    def sample_reuse(self) -> float:
        """sequences consumed / sequences produced"""
        return self.consumed / max(1, self.buf.pushed)
