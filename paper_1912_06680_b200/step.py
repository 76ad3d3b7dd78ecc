"""PPOOptimizer: composes one PPO optimizer step (§3.2) from the C-ABI calls.

    ppo_gae -> lstm_bptt_fwd -> ppo_loss_grad -> lstm_bptt_bwd -> grad_allreduce -> adam_step

PyTorch only provides device memory, streams and the process group that carries the NCCL
unique id; every step of the path runs in libppo5's kernels.
"""
from __future__ import annotations

import torch

from . import _lib as L

#: factorised heads, P:303-368 [App. Action Space]
HEAD_SIZES = (30, 4, 189, 189, 81, 81, 81)

#: Baseline hyperparameters, Table hyperparams; DESIGN Q3/Q4.
DEFAULT_HYPER = dict(T_step=4.0 / 30.0, horizon_s=180.0, lam=0.95, clip_eps=0.2, c_v=1.0,
                     c_e=0.01, lr=5e-5, beta1=0.9, beta2=0.999, adam_eps=1e-8, clip_sigma=5.0,
                     # NEXT-4 aux heads (DESIGN Q25/Q26; the paper gives no values)
                     c_win=1.0, c_rank=1.0, c_bld=1.0, aux_win_trunk=0.01, aux_horizon_s=120.0)


def _aligned_empty(nbytes: int, device, align: int = 1024) -> torch.Tensor:
    raw = torch.empty(nbytes + align, dtype=torch.uint8, device=device)
    off = (-raw.data_ptr()) % align
    return raw[off:off + nbytes]


class PPOOptimizer:
    """Owns theta (fp32 master, flat layout of ppo5.h), its bf16 shadow, Adam moments, the
    gradient buffer and the activation workspace for one rank's minibatch of B sequences."""

    def __init__(self, D: int, H: int, B: int, T: int = 16, head_sizes=HEAD_SIZES,
                 precision: str = "bf16", device="cuda", hyper: dict | None = None,
                 comm=None, n_buckets: int = 1, n_ws: int = 1, aux=(0, 0, 0),
                 dp: str = "allreduce", overlap: bool = True):
        self.D, self.H, self.B, self.T = D, H, B, T
        self.head_sizes = tuple(head_sizes)
        self.aux = tuple(aux)           # NEXT-4 (n_win, n_rank, n_bld) heads after the value
        self.A = sum(self.head_sizes) + 1 + sum(self.aux)
        self.bf16 = precision == "bf16"
        self.device = torch.device(device)
        self.hyper = dict(DEFAULT_HYPER, **(hyper or {}))
        self.dims = L.make_dims(D, H, T, self.head_sizes,
                                L.PPO_PREC_BF16 if self.bf16 else L.PPO_PREC_FP32, self.aux,
                                self.hyper["aux_win_trunk"] if sum(self.aux) else 0.0)
        self.layout = L.param_layout(self.dims)
        n = self.layout.n_total
        dev = self.device
        f32 = dict(dtype=torch.float32, device=dev)
        # dp = "fused" (with a comm): a9+a10 as one NVLink peer-memory kernel per rank
        # (ppo_dp_adam_step); m, v (and theta, when the bf16 shadow is what is all-gathered)
        # are then sharded, padded to world x shard for the in-place all-gather that brings
        # them up to date for a checkpoint
        if dp not in ("allreduce", "fused", "fused-push"):
            raise ValueError("dp must be 'allreduce', 'fused' or 'fused-push'")
        self.dp = "fused" if comm is not None and dp.startswith("fused") else "allreduce"
        world = 1
        if self.dp == "fused":
            import torch.distributed as dist
            world = dist.get_world_size() if dist.is_initialized() else 1
        n_mv = world * L.dp_shard(n, world) if self.dp == "fused" else n
        self._theta_full = torch.zeros(n_mv, **f32)
        self.theta = self._theta_full[:n]
        self._m_full = torch.zeros(n_mv, **f32)
        self._v_full = torch.zeros(n_mv, **f32)
        self.m = self._m_full[:n]
        self.v = self._v_full[:n]
        self.grad = torch.zeros(n, **f32)
        self.shadow = torch.zeros(n, dtype=torch.bfloat16, device=dev) if self.bf16 else None
        # "fused-push": the backward's epilogues deliver the gradient shards to their owners
        # over NVLink (bf16 path without the win-head trunk route); "fused" (pull): the owners
        # read them after the backward -- the default, 1-1.5% faster per step in the A/B
        self.dp_push = (self.dp == "fused" and dp == "fused-push" and world > 1 and self.bf16
                        and sum(self.aux) == 0)
        if self.dp == "fused":
            L.dp_attach(comm, self.grad, self.theta, self.shadow, n)
        # pull mode at world > 1: exchange W_xh_aug (97% of theta) on a second stream while the
        # backward's last GEMM (dW_o) still runs (lstm_bptt_bwd_ev + ppo_dp_adam_step_range)
        self._overlap = self.dp == "fused" and world > 1 and not self.dp_push and overlap
        if self._overlap:
            self._comm_stream = torch.cuda.Stream(device=dev)
            self._wxh_ev = torch.cuda.Event()
            self._xch_done = torch.cuda.Event()
            self._wxh_ev.record()        # (creates the events before the library records them)
            self._xch_done.record()
        # activation workspaces; n_ws = 2 lets the next step's x be uploaded into one while
        # the current step runs in the other
        self.ws_list = [_aligned_empty(L.ws_bytes(self.dims, B), dev) for _ in range(n_ws)]
        self.ws = self.ws_list[0]
        act_dtype = torch.bfloat16 if self.bf16 else torch.float32
        rows = T * B
        self.out = torch.empty(rows, self.A, **f32)
        self.dout = torch.empty(rows, self.A, dtype=act_dtype, device=dev)
        self.logp = torch.empty(rows, **f32)
        self.stats = torch.zeros(L.PPO_STATS_BUF, **f32)
        self.adv = torch.empty(T, B, **f32)
        self.ret = torch.empty(T, B, **f32)
        self.t = 0
        # graph mode (capture()): the Adam step number lives on the device (adam_step_ctr):
        # int64 steps taken + a float scratch, 16-byte aligned
        self.device_t = False
        self._ctr = torch.zeros(2, dtype=torch.int64, device=dev)
        self.comm = comm
        self.n_buckets = n_buckets
        h = self.hyper
        self.gamma = 1.0 - h["T_step"] / h["horizon_s"]  # Eq. horizon
        self.loss_cfg = L.ppo_loss_cfg(h["clip_eps"], h["c_v"], h["c_e"], 0.0, h["c_win"],
                                       h["c_rank"], h["c_bld"])

    # ---------------------------------------------------------------- parameters
    @property
    def weights(self):
        """the tensor the GEMMs read: bf16 shadow or fp32 theta"""
        return self.shadow if self.bf16 else self.theta

    def load_canonical(self, Wx, Wh, b, Wo, bo, stream=None):
        """canonical fp32 device tensors (gate blocks [i;f;g;o]) -> theta (+ bf16 shadow)"""
        L.ppo_pack_params(self.dims, Wx, Wh, b, Wo, bo, self.theta, stream)
        if self.bf16:
            L.ppo_cast_bf16(self.theta, self.shadow, stream)

    def unpack(self, flat: torch.Tensor, stream=None) -> dict:
        """flat theta-layout vector (params or grads) -> canonical fp32 tensors"""
        H, D, A = self.H, self.D, self.A
        f32 = dict(dtype=torch.float32, device=self.device)
        out = dict(Wx=torch.empty(4 * H, D, **f32), Wh=torch.empty(4 * H, H, **f32),
                   b=torch.empty(4 * H, **f32), Wo=torch.empty(A, H, **f32), bo=torch.empty(A, **f32))
        L.ppo_unpack_params(self.dims, flat, out["Wx"], out["Wh"], out["b"], out["Wo"], out["bo"],
                            stream)
        return out

    # ---------------------------------------------------------------- checkpoint / resume
    def state_dict(self) -> dict:
        """fp32 parameters and Adam moments in the canonical layout (gate blocks [i;f;g;o],
        separate W_x, W_h, b, W_o, b_o: the oracle's), the Adam step t and the shapes; host
        tensors, loadable into an optimizer of the same dims.  Collective when
        dp = "fused" (the sharded moments are all-gathered first)."""
        self.gather_sharded()
        torch.cuda.synchronize(self.device)
        cpu = lambda d: {k: v.cpu() for k, v in d.items()}  # noqa: E731
        return {"format": "ppo5-ckpt-1", "t": self.sync_t(), "D": self.D, "H": self.H,
                "head_sizes": list(self.head_sizes), "aux": list(self.aux),
                "params": cpu(self.unpack(self.theta)), "m": cpu(self.unpack(self.m)),
                "v": cpu(self.unpack(self.v))}

    def load_state_dict(self, sd: dict, stream=None):
        if sd.get("format") != "ppo5-ckpt-1":
            raise ValueError("not a ppo5 checkpoint")
        if (sd["D"], sd["H"], tuple(sd["head_sizes"]), tuple(sd["aux"])) != \
                (self.D, self.H, self.head_sizes, self.aux):
            raise ValueError("checkpoint shapes differ from this optimizer's")
        names = ("Wx", "Wh", "b", "Wo", "bo")
        for key, flat in (("params", self.theta), ("m", self.m), ("v", self.v)):
            t = [sd[key][k].to(self.device, torch.float32).contiguous() for k in names]
            L.ppo_pack_params(self.dims, *t, flat, stream)
        if self.bf16:
            L.ppo_cast_bf16(self.theta, self.shadow, stream)
        self.t = int(sd["t"])
        self._ctr[0] = self.t

    def save(self, path: str):
        torch.save(self.state_dict(), path)

    def load(self, path: str):
        self.load_state_dict(torch.load(path, map_location="cpu"))

    # ---------------------------------------------------------------- zero-copy inputs
    def select_ws(self, i: int):
        """make workspace i the one the next forward/backward use"""
        self.ws = self.ws_list[i]

    def put_x(self, x: torch.Tensor, ws: int | None = None, stream=None):
        """copy x [T][B][D] (pinned host or device) straight into a workspace's x rows; the
        step then runs with batch["x"] = None (ppo_copy_x)"""
        L.ppo_copy_x(self.dims, self.B, x, self.ws if ws is None else self.ws_list[ws], stream)

    # ---------------------------------------------------------------- the step
    def gae(self, batch, stream=None):
        """a1: advantages/returns written time-major [T][B] for the minibatch.  The rollouts
        must cover exactly this optimizer's B sequences: rew, done [R][L], val [R][L+1],
        L % T == 0 and R * L / T == B (ppo_gae writes R*L advantages)."""
        h = self.hyper
        rew, val, done = batch["rew"], batch["val"], batch["done"]
        if rew.dim() != 2 or tuple(done.shape) != tuple(rew.shape):
            raise ValueError(f"rew and done must both be [R][L]; got {tuple(rew.shape)}, "
                             f"{tuple(done.shape)}")
        R, Lr = rew.shape
        if tuple(val.shape) != (R, Lr + 1):
            raise ValueError(f"val must be [R][L+1] = {(R, Lr + 1)}; got {tuple(val.shape)}")
        if Lr % self.T or R * (Lr // self.T) != self.B:
            raise ValueError(f"rollouts [{R}][{Lr}] do not hold exactly B = {self.B} sequences "
                             f"of T = {self.T} steps")
        L.ppo_gae(batch["rew"], batch["val"], batch["done"], self.gamma, h["lam"], self.adv,
                  self.ret, seq_T=self.T, stream=stream)

    def aux_labels(self, batch, stream=None):
        """NEXT-4: aux-head targets of the minibatch from its segments' aux inputs (last,
        outcome, rank, events, boot; DESIGN Q27), into batch["aux_label"] [T][B][n_aux]"""
        if "aux_label" not in batch or batch["aux_label"] is None:
            batch["aux_label"] = torch.empty(self.T, self.B, sum(self.aux), device=self.device)
        h = self.hyper
        g2 = 1.0 - h["T_step"] / h["aux_horizon_s"]     # 2-minute horizon
        L.ppo_aux_labels(self.dims, batch["last"], batch["outcome"], batch["rank"],
                         batch["events"], batch["boot"], g2, batch["aux_label"], seq_T=self.T,
                         stream=stream)

    def forward_streamed(self, batch, x_events, stream=None):
        """a2-a4 with x arriving in the workspace slice by slice (ppo_copy_x_slice): step t
        waits on x_events[t] (lstm_bptt_fwd_ev)"""
        L.lstm_bptt_fwd_ev(self.dims, self.weights, batch["h0"], batch["c0"], self.B, self.ws,
                           self.out, x_events, stream)

    def step_streamed(self, batch, x_events, rest_event, stream=None, dx=None):
        """The step with host inputs still streaming in: GAE and the forward start as soon as
        their inputs land (x per time step); the loss waits on rest_event (act, head_on,
        avail, logp_old ...)."""
        import torch
        self.gae(batch, stream)
        if sum(self.aux) and "events" in batch:
            self.aux_labels(batch, stream)
        self.forward_streamed(batch, x_events, stream)
        (stream or torch.cuda.current_stream()).wait_event(rest_event)
        self.loss(batch, stream=stream)
        self.backward(stream)
        if dx is not None:
            self.input_grad(dx, stream)
        self.allreduce(stream)
        self.apply(stream)
        return self.stats[:L.PPO_STATS]

    def forward(self, batch, stream=None):
        """a2-a4; batch["x"] None = x already in the workspace (put_x / ppo_gather)"""
        L.lstm_bptt_fwd(self.dims, self.weights, batch.get("x"), batch["h0"], batch["c0"], self.B,
                        self.ws, self.out, stream)

    def loss(self, batch, logp_old=None, stream=None):
        """a5"""
        L.ppo_loss_grad(self.dims, self.out, batch["act"], batch["head_on"], batch["avail"],
                        batch["logp_old"] if logp_old is None else logp_old, self.adv, self.ret,
                        batch.get("valid"), self.B, self.loss_cfg, self.dout, self.logp,
                        self.stats, stream, aux_label=batch.get("aux_label"))

    def backward(self, stream=None):
        """a6-a8 (dp push mode: + the reduce-scatter of the final weight gradients)"""
        if self.dp_push:
            L.lstm_bptt_bwd_dp(self.dims, self.weights, self.ws, self.dout, self.B, self.grad,
                               self.comm, stream)
            return
        if self._overlap:
            L.lstm_bptt_bwd_ev(self.dims, self.weights, self.ws, self.dout, self.B, self.grad,
                               self._wxh_ev, stream)
            return
        L.lstm_bptt_bwd(self.dims, self.weights, self.ws, self.dout, self.B, self.grad, stream)

    def input_grad(self, dx: torch.Tensor, stream=None):
        """NEXT-4: dL/dx [T][B][D] fp32 for the observation-processing network (after backward)"""
        L.lstm_input_grad(self.dims, self.weights, self.ws, self.B, dx, stream)

    def allreduce(self, stream=None):
        """a9 (dp = "fused": folded into apply)"""
        if self.comm is not None and self.dp == "allreduce":
            L.grad_allreduce(self.comm, self.grad, self.n_buckets, stream)

    def apply(self, stream=None):
        """a10 (dp = "fused": a9 + a10 on this rank's shard, theta and shadow all-gathered)"""
        h = self.hyper
        self.t += 1
        if self.device_t:
            L.adam_step_ctr(self.theta, self.shadow, self.grad, self.m, self.v, self._ctr, h["lr"],
                            h["beta1"], h["beta2"], h["adam_eps"], h["clip_sigma"], stream)
            return
        if self.dp == "fused" and self._overlap:
            # W_xh_aug's shard exchange + Adam on the comm stream once its gradient is final
            # (overlapping dW_o), then W_o_aug's on this stream; the next step waits for both
            cs = self._comm_stream
            main = stream or torch.cuda.current_stream(self.device)
            off = self.layout.off_wo
            args = (self.t, h["lr"], h["beta1"], h["beta2"], h["adam_eps"], h["clip_sigma"])
            cs.wait_event(self._wxh_ev)
            L.dp_adam_step_range(self.comm, self.m, self.v, *args, 0, off, stream=cs)
            L.dp_adam_step_range(self.comm, self.m, self.v, *args, off, self.layout.n_total,
                                 stream=main)
            self._xch_done.record(cs)
            main.wait_event(self._xch_done)
            return
        if self.dp == "fused":
            L.dp_adam_step(self.comm, self.m, self.v, self.t, h["lr"], h["beta1"], h["beta2"],
                           h["adam_eps"], h["clip_sigma"], staged=self.dp_push, stream=stream)
            return
        L.adam_step(self.theta, self.shadow, self.grad, self.m, self.v, self.t, h["lr"],
                    h["beta1"], h["beta2"], h["adam_eps"], h["clip_sigma"], stream)

    def gather_sharded(self, stream=None):
        """dp = "fused": bring every rank's m, v (and theta, on the bf16 path) up to date from
        the owners' shards (collective; state_dict calls it)"""
        if self.dp == "fused":
            L.dp_allgather(self.comm, self._m_full, stream)
            L.dp_allgather(self.comm, self._v_full, stream)
            if self.bf16:
                L.dp_allgather(self.comm, self._theta_full, stream)

    def step(self, batch, stream=None, dx=None):
        """One full optimizer step a1-a10 on this rank; returns the device stats tensor.
        dx: optional [T][B][D] fp32 output for dL/dx (NEXT-4)."""
        self.gae(batch, stream)
        if sum(self.aux) and "events" in batch:
            self.aux_labels(batch, stream)
        self.forward(batch, stream)
        self.loss(batch, stream=stream)
        self.backward(stream)
        if dx is not None:
            self.input_grad(dx, stream)
        self.allreduce(stream)
        self.apply(stream)
        return self.stats[:L.PPO_STATS]

    # ---------------------------------------------------------------- CUDA graphs
    def use_device_t(self):
        """Switch Adam to the device step counter (adam_step_ctr), continuing from self.t.
        (Single rank or NCCL-allreduce exchange: the fused exchange takes t from the host.)"""
        if self.dp == "fused":
            raise ValueError("the device step counter needs dp='allreduce' (or one rank)")
        if not self.device_t:
            self._ctr[0] = self.t
            self.device_t = True

    def sync_t(self) -> int:
        """host copy of the step count (graph replays advance only the device counter)"""
        if self.device_t:
            self.t = int(self._ctr[0].item())
        return self.t

    def capture(self, batch, dx=None) -> "torch.cuda.CUDAGraph":
        """Capture one whole optimizer step a1-a10 on `batch` (its tensors stay the step's
        inputs: refill them in place between replays) into a CUDA graph; each replay() is one
        step (the step's ~100 launches cost one graph launch).  Adam then
        takes its step number from the device counter.  Run at least one eager step() first
        (kernel attributes and modules are set up outside the capture).  Single-rank or
        NCCL-allreduce exchange only (the fused exchange's IPC barriers are not captured)."""
        if self.dp == "fused":
            raise ValueError("capture(): the fused DP exchange is not graph-capturable; "
                             "use dp='allreduce'")
        self.use_device_t()
        t_host = self.t
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step(batch, dx=dx)
        self.t = t_host           # capturing records the launches, it does not run them
        return g

    def current_logp(self, batch, stream=None) -> torch.Tensor:
        """log pi_theta(a) for the batch (forward + loss pass); used to synthesise behaviour
        log-probs like the forward-pass GPUs'."""
        self.gae(batch, stream)
        if sum(self.aux) and "events" in batch:
            self.aux_labels(batch, stream)
        self.forward(batch, stream)
        self.loss(batch, logp_old=torch.zeros_like(self.logp), stream=stream)
        return self.logp.view(self.T, self.B).clone()
