"""Thin ctypes binding of libppo5.so (include/ppo5.h).  Argument marshalling only: every step
of the PPO path runs in the library's CUDA kernels.  Names follow the C ABI.

Raises ImportError at import time if the in-tree library has not been built -- there is no
fallback of any kind.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_size_t, c_uint8, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libppo5.so")
# A/B timing of two builds (tools/ab_builds.sh): load another build of the same ABI
if os.environ.get("PPO_LIB_PATH"):
    LIB_PATH = os.environ["PPO_LIB_PATH"]

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python paper_1912_06680_b200/build.py` "
                      "(or __graft_entry__.build()).  There is no CPU fallback.")

import torch  # noqa: E402,F401  -- load torch (and its NCCL) before libppo5 links against it

_lib = ctypes.CDLL(LIB_PATH)

PPO_OK, PPO_E_ARG, PPO_E_SHAPE, PPO_E_ALIGN, PPO_E_CUDA, PPO_E_NCCL, PPO_E_UNSUPPORTED = (
    0, -1, -2, -3, -4, -5, -6)
PPO_PREC_BF16, PPO_PREC_FP32 = 0, 1
PPO_MAX_HEADS = 8
PPO_STATS = 9
PPO_LOSS_BLOCKS = 1184
PPO_STATS_BUF = PPO_STATS * (1 + PPO_LOSS_BLOCKS)
PPO_COMM_ID_BYTES = 128
STAT_NAMES = ("loss", "pg", "vf", "ent", "approx_kl", "clipfrac", "n_valid", "flags", "aux")


class ppo_dims(ctypes.Structure):
    _fields_ = [("D", c_int32), ("H", c_int32), ("T", c_int32), ("n_heads", c_int32),
                ("head_sizes", c_int32 * PPO_MAX_HEADS), ("precision", c_int32),
                ("n_aux_win", c_int32), ("n_aux_rank", c_int32), ("n_aux_bld", c_int32),
                ("aux_win_trunk", c_float)]


class ppo_param_layout(ctypes.Structure):
    _fields_ = [("Kx", c_int64), ("Ko", c_int64), ("A", c_int64), ("off_wxh", c_int64),
                ("n_wxh", c_int64), ("off_wo", c_int64), ("n_wo", c_int64), ("n_total", c_int64)]


class ppo_loss_cfg(ctypes.Structure):
    _fields_ = [("clip_eps", c_float), ("c_v", c_float), ("c_e", c_float), ("denom", c_float),
                ("c_win", c_float), ("c_rank", c_float), ("c_bld", c_float)]


class ppo_prof_entry(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", c_int32), ("total_ms", c_double)]


class ppo_buffer(ctypes.Structure):
    _fields_ = [("x", c_void_p), ("h0", c_void_p), ("c0", c_void_p), ("act", c_void_p),
                ("head_on", c_void_p), ("avail", c_void_p), ("logp_old", c_void_p),
                ("adv", c_void_p), ("ret", c_void_p), ("valid", c_void_p),
                ("capacity", c_int64)]


class ppo_reward_cfg(ctypes.Structure):
    _fields_ = [("tau", c_float), ("decay_base", c_float), ("decay_seconds", c_float),
                ("step_seconds", c_float), ("zero_sum", c_int32)]


class PPOError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libppo5 error {code}: {msg}")
        self.code = code


def _sig(name, args, res=c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res
    return f


_D = POINTER(ppo_dims)
_lib_fns = dict(
    ppo_last_error=([], c_char_p),
    ppo_version=([], c_char_p),
    ppo_get_param_layout=([_D, POINTER(ppo_param_layout)], c_int),
    ppo_pack_params=([_D] + [c_void_p] * 7, c_int),
    ppo_unpack_params=([_D] + [c_void_p] * 7, c_int),
    ppo_cast_bf16=([c_void_p, c_void_p, c_size_t, c_void_p], c_int),
    ppo_gae_scratch_bytes=([c_int64, c_int64, POINTER(c_size_t)], c_int),
    ppo_gae=([c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_float, c_float, c_int32, c_void_p,
              c_void_p, c_void_p, c_size_t, c_void_p], c_int),
    lstm_ws_bytes=([_D, c_int64, POINTER(c_size_t)], c_int),
    lstm_bptt_fwd=([_D, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_size_t,
                    c_void_p, c_void_p], c_int),
    lstm_ws_x=([_D, c_int64, c_void_p, POINTER(c_void_p), POINTER(c_int64)], c_int),
    ppo_copy_x_slice=([_D, c_int64, c_int32, c_void_p, c_int64, c_void_p, c_size_t, c_void_p],
                      c_int),
    lstm_bptt_fwd_ev=([_D, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_size_t, c_void_p,
                       POINTER(c_void_p), c_void_p], c_int),
    ppo_copy_x=([_D, c_int64, c_void_p, c_int64, c_void_p, c_size_t, c_void_p], c_int),
    ppo_loss_grad=([_D] + [c_void_p] * 9 + [c_int64, POINTER(ppo_loss_cfg), c_void_p, c_void_p,
                                             c_void_p, c_void_p], c_int),
    ppo_aux_labels=([_D, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                     c_float, c_int32, c_void_p, c_void_p], c_int),
    lstm_bptt_bwd=([_D, c_void_p, c_void_p, c_size_t, c_void_p, c_int64, c_void_p, c_void_p], c_int),
    ppo_comm_unique_id=([POINTER(c_uint8)], c_int),
    ppo_comm_init=([POINTER(c_uint8), c_int, c_int, POINTER(c_void_p)], c_int),
    grad_allreduce=([c_void_p, c_void_p, c_size_t, c_int32, c_void_p], c_int),
    ppo_comm_destroy=([c_void_p], c_int),
    ppo_dp_shard=([c_size_t, c_int], c_size_t),
    ppo_dp_attach=([c_void_p, c_void_p, c_void_p, c_void_p, c_size_t], c_int),
    ppo_dp_adam_step=([c_void_p, c_void_p, c_void_p, c_int64, c_double, c_double, c_double,
                       c_double, c_double, c_int32, c_void_p], c_int),
    lstm_bptt_bwd_dp=([_D, c_void_p, c_void_p, c_size_t, c_void_p, c_int64, c_void_p, c_void_p,
                       c_void_p], c_int),
    ppo_dp_allgather=([c_void_p, c_void_p, c_void_p], c_int),
    ppo_dp_adam_step_range=([c_void_p, c_void_p, c_void_p, c_int64, c_double, c_double, c_double,
                             c_double, c_double, c_int32, c_size_t, c_size_t, c_void_p], c_int),
    lstm_bptt_bwd_ev=([_D, c_void_p, c_void_p, c_size_t, c_void_p, c_int64, c_void_p, c_void_p,
                       c_void_p], c_int),
    ppo_test_dp_adam=([c_int32] + [POINTER(c_void_p)] * 6 + [c_size_t, c_int64, c_double,
                      c_double, c_double, c_double, c_double, c_void_p], c_int),
    adam_step=([c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_int64, c_double,
                c_double, c_double, c_double, c_double, c_void_p], c_int),
    adam_step_ctr=([c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p,
                    c_double, c_double, c_double, c_double, c_double, c_void_p], c_int),
    ppo_sample_indices=([c_int64, c_int64, ctypes.c_uint64, ctypes.c_uint64, c_void_p, c_void_p], c_int),
    ppo_gather=([_D, POINTER(ppo_buffer), c_void_p, c_int64, c_void_p, c_size_t] + [c_void_p] * 8,
                c_int),
    ppo_reward_gae_scratch_bytes=([POINTER(c_size_t)], c_int),
    ppo_reward_gae=([c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p,
                     POINTER(ppo_reward_cfg), c_void_p, c_float, c_float, c_int32, c_void_p,
                     c_void_p, c_void_p, c_void_p, c_size_t, c_void_p], c_int),
    lstm_input_grad=([_D, c_void_p, c_void_p, c_size_t, c_int64, c_void_p, c_void_p], c_int),
    ppo_infer_step_ctr=([_D, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                         ctypes.c_uint64, c_void_p, ctypes.c_uint32, c_int64, c_void_p, c_size_t,
                         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p], c_int),
    ppo_infer_ws_bytes=([_D, c_int64, POINTER(c_size_t)], c_int),
    ppo_infer_weights_bytes=([_D, POINTER(c_size_t)], c_int),
    ppo_infer_pack_weights=([_D, c_void_p, c_void_p, c_size_t, c_void_p], c_int),
    ppo_infer_step=([_D, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                     ctypes.c_uint64, ctypes.c_uint64, c_int64, c_void_p, c_size_t, c_void_p, c_void_p, c_void_p,
                     c_void_p, c_void_p, c_void_p], c_int),
    ppo_device_info=([POINTER(c_int32)] * 3, c_int),
    ppo_prof_start=([], c_int),
    ppo_prof_stop=([POINTER(ppo_prof_entry), c_int32, POINTER(c_int32)], c_int),
    ppo_test_tc_gemm=([c_int, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p], c_int),
)
EXPORTED = tuple(_lib_fns)
for _n, (_a, _r) in _lib_fns.items():
    if os.environ.get("PPO_LIB_PATH") and not hasattr(_lib, _n):
        continue   # A/B against an older build: calls it lacks are unavailable
    _sig(_n, _a, _r)


def last_error() -> str:
    return _lib.ppo_last_error().decode()


def version() -> str:
    return _lib.ppo_version().decode()


def _check(rc):
    if rc != PPO_OK:
        raise PPOError(rc, last_error())


# ------------------------------------------------------------------ marshalling helpers
def _p(t):
    """device/host pointer of a torch tensor (or None -> NULL)."""
    return None if t is None else c_void_p(t.data_ptr())


def _s(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return c_void_p(stream.cuda_stream)


def make_dims(D, H, T, head_sizes, precision=PPO_PREC_BF16, aux=(0, 0, 0),
              win_trunk=0.0) -> ppo_dims:
    d = ppo_dims()
    d.D, d.H, d.T = D, H, T
    d.n_heads = len(head_sizes)
    for i, h in enumerate(head_sizes):
        d.head_sizes[i] = h
    d.precision = precision
    d.n_aux_win, d.n_aux_rank, d.n_aux_bld = aux
    d.aux_win_trunk = win_trunk
    return d


def param_layout(dims: ppo_dims) -> ppo_param_layout:
    out = ppo_param_layout()
    _check(_lib.ppo_get_param_layout(ctypes.byref(dims), ctypes.byref(out)))
    return out


def ws_bytes(dims: ppo_dims, B: int) -> int:
    n = c_size_t()
    _check(_lib.lstm_ws_bytes(ctypes.byref(dims), B, ctypes.byref(n)))
    return n.value


# ------------------------------------------------------------------ the hot-path calls
def ppo_pack_params(dims, Wx, Wh, b, Wo, bo, theta, stream=None):
    _check(_lib.ppo_pack_params(ctypes.byref(dims), _p(Wx), _p(Wh), _p(b), _p(Wo), _p(bo),
                                _p(theta), _s(stream)))


def ppo_unpack_params(dims, theta, Wx, Wh, b, Wo, bo, stream=None):
    _check(_lib.ppo_unpack_params(ctypes.byref(dims), _p(theta), _p(Wx), _p(Wh), _p(b), _p(Wo),
                                  _p(bo), _s(stream)))


def ppo_cast_bf16(src, dst, stream=None):
    _check(_lib.ppo_cast_bf16(_p(src), _p(dst), src.numel(), _s(stream)))


def gae_scratch_bytes(R: int, L: int) -> int:
    n = c_size_t()
    _check(_lib.ppo_gae_scratch_bytes(R, L, ctypes.byref(n)))
    return n.value


def ppo_gae(rew, val, done, gamma, lam, adv, ret, seq_T=0, scratch=None, stream=None):
    """scratch: uint8 device tensor of >= gae_scratch_bytes(R, L) (None if that is 0)"""
    R, L = rew.shape
    nbytes = 0 if scratch is None else scratch.numel() * scratch.element_size()
    _check(_lib.ppo_gae(_p(rew), _p(val), _p(done), R, L, gamma, lam, seq_T, _p(adv), _p(ret),
                        _p(scratch), nbytes, _s(stream)))


def lstm_bptt_fwd(dims, w, x, h0, c0, B, ws, out, stream=None):
    """x = None: inputs already gathered into ws by ppo_gather"""
    _check(_lib.lstm_bptt_fwd(ctypes.byref(dims), _p(w), _p(x), _p(h0), _p(c0), B, _p(ws),
                              ws.numel() * ws.element_size(), _p(out), _s(stream)))


def lstm_ws_x(dims, B, ws):
    """-> (device address, row stride in elements) of x inside the workspace"""
    p, ld = c_void_p(), c_int64()
    _check(_lib.lstm_ws_x(ctypes.byref(dims), B, _p(ws), ctypes.byref(p), ctypes.byref(ld)))
    return p.value, ld.value


def ppo_copy_x(dims, B, src, ws, stream=None):
    """src: contiguous [T][B][D] tensor (pinned host or device)"""
    _check(_lib.ppo_copy_x(ctypes.byref(dims), B, _p(src), src.shape[-1], _p(ws),
                           ws.numel() * ws.element_size(), _s(stream)))


def ppo_copy_x_slice(dims, B, t, src, ws, stream=None):
    """src: [B][D] contiguous (pinned host or device): time slice t of x"""
    _check(_lib.ppo_copy_x_slice(ctypes.byref(dims), B, t, _p(src), src.shape[-1], _p(ws),
                                 ws.numel() * ws.element_size(), _s(stream)))


def lstm_bptt_fwd_ev(dims, w, h0, c0, B, ws, out, events, stream=None):
    """events: list of T torch.cuda.Event (or None entries)"""
    arr = (c_void_p * len(events))(*[None if e is None else c_void_p(e.cuda_event)
                                     for e in events])
    _check(_lib.lstm_bptt_fwd_ev(ctypes.byref(dims), _p(w), _p(h0), _p(c0), B, _p(ws),
                                 ws.numel() * ws.element_size(), _p(out), arr, _s(stream)))


def ppo_loss_grad(dims, out, act, head_on, avail, logp_old, adv, ret, valid, B, cfg, dout, logp,
                  stats, stream=None, aux_label=None):
    _check(_lib.ppo_loss_grad(ctypes.byref(dims), _p(out), _p(act), _p(head_on), _p(avail),
                              _p(logp_old), _p(adv), _p(ret), _p(valid), _p(aux_label), B,
                              ctypes.byref(cfg), _p(dout), _p(logp), _p(stats), _s(stream)))


def ppo_aux_labels(dims, last, outcome, rank, events, boot, gamma2, labels, seq_T=0,
                   stream=None):
    """NEXT-4 targets per segment: events [R][L][n_bld] (L from its shape)"""
    R, Lseg = events.shape[0], events.shape[1]
    _check(_lib.ppo_aux_labels(ctypes.byref(dims), R, Lseg, _p(last), _p(outcome), _p(rank),
                               _p(events), _p(boot), gamma2, seq_T, _p(labels), _s(stream)))


def lstm_bptt_bwd(dims, w, ws, dout, B, grad, stream=None):
    _check(_lib.lstm_bptt_bwd(ctypes.byref(dims), _p(w), _p(ws), ws.numel() * ws.element_size(),
                              _p(dout), B, _p(grad), _s(stream)))


def adam_step(p, p_bf16, g, m, v, t, lr, b1, b2, eps, clip_sigma, stream=None):
    _check(_lib.adam_step(_p(p), _p(p_bf16), _p(g), _p(m), _p(v), p.numel(), t, lr, b1, b2, eps,
                          clip_sigma, _s(stream)))


def adam_step_ctr(p, p_bf16, g, m, v, ctr, lr, b1, b2, eps, clip_sigma, stream=None):
    """ctr: int64 device tensor of >= 2 elements, 16-byte aligned (steps taken; scratch)"""
    _check(_lib.adam_step_ctr(_p(p), _p(p_bf16), _p(g), _p(m), _p(v), p.numel(), _p(ctr), lr, b1,
                              b2, eps, clip_sigma, _s(stream)))


def make_buffer(t: dict, capacity: int) -> ppo_buffer:
    """ppo_buffer view of a dict of device tensors (keys as in the struct)"""
    b = ppo_buffer()
    for k in ("x", "h0", "c0", "act", "head_on", "avail", "logp_old", "adv", "ret", "valid"):
        setattr(b, k, None if t.get(k) is None else t[k].data_ptr())
    b.capacity = capacity
    return b


def ppo_sample_indices(capacity, B, seed, step, idx, stream=None):
    _check(_lib.ppo_sample_indices(capacity, B, seed, step, _p(idx), _s(stream)))


def ppo_gather(dims, buf: ppo_buffer, idx, B, ws, act, head_on, avail, logp_old, adv, ret, valid,
               stream=None):
    _check(_lib.ppo_gather(ctypes.byref(dims), ctypes.byref(buf), _p(idx), B, _p(ws),
                           ws.numel() * ws.element_size(), _p(act), _p(head_on), _p(avail),
                           _p(logp_old), _p(adv), _p(ret), _p(valid), _s(stream)))


def reward_gae_scratch_bytes() -> int:
    n = c_size_t()
    _check(_lib.ppo_reward_gae_scratch_bytes(ctypes.byref(n)))
    return n.value


def ppo_reward_gae(shaped, win, step0, val, done, cfg, stats, gamma, lam, adv, ret, scratch,
                   seq_T=0, rew_out=None, stream=None):
    G, _, Lr = shaped.shape
    _check(_lib.ppo_reward_gae(_p(shaped), _p(win), _p(step0), G, Lr, _p(val), _p(done),
                               ctypes.byref(cfg), _p(stats), gamma, lam, seq_T, _p(rew_out),
                               _p(adv), _p(ret), _p(scratch),
                               scratch.numel() * scratch.element_size(), _s(stream)))


def lstm_input_grad(dims, w, ws, B, dx, stream=None):
    _check(_lib.lstm_input_grad(ctypes.byref(dims), _p(w), _p(ws), ws.numel() * ws.element_size(),
                                B, _p(dx), _s(stream)))


def infer_ws_bytes(dims, B) -> int:
    n = c_size_t()
    _check(_lib.ppo_infer_ws_bytes(ctypes.byref(dims), B, ctypes.byref(n)))
    return n.value


def infer_weights_bytes(dims) -> int:
    n = c_size_t()
    _check(_lib.ppo_infer_weights_bytes(ctypes.byref(dims), ctypes.byref(n)))
    return n.value


def ppo_infer_pack_weights(dims, w, wt, stream=None):
    _check(_lib.ppo_infer_pack_weights(ctypes.byref(dims), _p(w), _p(wt),
                                       wt.numel() * wt.element_size(), _s(stream)))


def ppo_infer_step(dims, w, x, h, c, avail, head_table, seed, step, B, ws, act, head_on, logp,
                   value=None, out=None, stream=None):
    _check(_lib.ppo_infer_step(ctypes.byref(dims), _p(w), _p(x), _p(h), _p(c), _p(avail),
                               _p(head_table), seed, step, B, _p(ws),
                               ws.numel() * ws.element_size(), _p(act), _p(head_on), _p(logp),
                               _p(value), _p(out), _s(stream)))


PPO_INFER_STATE_CURRENT = 1


def ppo_infer_step_ctr(dims, w, x, h, c, avail, head_table, seed, step_ctr, B, ws, act, head_on,
                       logp, value=None, out=None, stream=None, flags=0):
    """step_ctr: device int64 tensor [1] (steps taken so far; advanced by the call)"""
    _check(_lib.ppo_infer_step_ctr(ctypes.byref(dims), _p(w), _p(x), _p(h), _p(c), _p(avail),
                                   _p(head_table), seed, _p(step_ctr), flags, B, _p(ws),
                                   ws.numel() * ws.element_size(), _p(act), _p(head_on),
                                   _p(logp), _p(value), _p(out), _s(stream)))


def comm_unique_id() -> bytes:
    buf = (c_uint8 * PPO_COMM_ID_BYTES)()
    _check(_lib.ppo_comm_unique_id(buf))
    return bytes(buf)


def comm_init(uid: bytes, rank: int, world: int) -> c_void_p:
    buf = (c_uint8 * PPO_COMM_ID_BYTES).from_buffer_copy(uid)
    h = c_void_p()
    _check(_lib.ppo_comm_init(buf, rank, world, ctypes.byref(h)))
    return h


def grad_allreduce(comm, g, n_buckets=1, stream=None):
    _check(_lib.grad_allreduce(comm, _p(g), g.numel(), n_buckets, _s(stream)))


def comm_destroy(comm):
    _check(_lib.ppo_comm_destroy(comm))


def dp_shard(n: int, world: int) -> int:
    """floats per rank shard of the fused a9+a10 path (a multiple of 64)"""
    return int(_lib.ppo_dp_shard(n, world))


def dp_attach(comm, g, p, p_bf16, n: int):
    """collective: map every rank's grad / theta / shadow for ppo_dp_adam_step"""
    _check(_lib.ppo_dp_attach(comm, _p(g), _p(p), _p(p_bf16), n))


def dp_adam_step(comm, m, v, t, lr, b1, b2, eps, clip_sigma, staged=False, stream=None):
    _check(_lib.ppo_dp_adam_step(comm, _p(m), _p(v), t, lr, b1, b2, eps, clip_sigma,
                                 1 if staged else 0, _s(stream)))


def dp_adam_step_range(comm, m, v, t, lr, b1, b2, eps, clip_sigma, lo, hi, staged=False,
                       stream=None):
    _check(_lib.ppo_dp_adam_step_range(comm, _p(m), _p(v), t, lr, b1, b2, eps, clip_sigma,
                                       1 if staged else 0, lo, hi, _s(stream)))


def lstm_bptt_bwd_ev(dims, w, ws, dout, B, grad, wxh_ready=None, stream=None):
    """backward recording wxh_ready (torch.cuda.Event) once the W_xh gradient is final"""
    _check(_lib.lstm_bptt_bwd_ev(ctypes.byref(dims), _p(w), _p(ws), ws.numel() * ws.element_size(),
                                 _p(dout), B, _p(grad),
                                 None if wxh_ready is None else c_void_p(wxh_ready.cuda_event),
                                 _s(stream)))


def lstm_bptt_bwd_dp(dims, w, ws, dout, B, grad, comm, stream=None):
    """backward that also pushes the final weight gradients to the DP owners' staging"""
    _check(_lib.lstm_bptt_bwd_dp(ctypes.byref(dims), _p(w), _p(ws), ws.numel() * ws.element_size(),
                                 _p(dout), B, _p(grad), comm, _s(stream)))


def dp_allgather(comm, buf, stream=None):
    _check(_lib.ppo_dp_allgather(comm, _p(buf), _s(stream)))


def test_dp_adam(g, p, p_bf16, m, v, t, lr, b1, b2, eps, clip_sigma, stage=None, stream=None):
    """the fused a9+a10 kernel for len(g) virtual ranks on this device (lists of tensors;
    p_bf16 / stage None = fp32 path / pull mode)"""
    W = len(g)

    def arr(ts):
        return None if ts is None else (c_void_p * W)(*[t.data_ptr() for t in ts])
    _check(_lib.ppo_test_dp_adam(W, arr(g), arr(p), arr(p_bf16), arr(m), arr(v), arr(stage),
                                 g[0].numel(), t, lr, b1, b2, eps, clip_sigma, _s(stream)))


def device_info() -> dict:
    """{'sms', 'die0_sms', 'die1_sms'} of the current device (die split 0/0 = none found)"""
    a, b, c = c_int32(), c_int32(), c_int32()
    _check(_lib.ppo_device_info(ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return {"sms": a.value, "die0_sms": b.value, "die1_sms": c.value}


def prof_start():
    _check(_lib.ppo_prof_start())


def prof_stop(max_entries: int = 64) -> dict:
    """-> {kernel tag: (launches, total device ms)} recorded since prof_start()"""
    arr = (ppo_prof_entry * max_entries)()
    n = c_int32()
    _check(_lib.ppo_prof_stop(arr, max_entries, ctypes.byref(n)))
    return {arr[i].name.decode(): (arr[i].launches, arr[i].total_ms)
            for i in range(min(n.value, max_entries))}


def test_tc_gemm(mode, A, B, C, M, N, K, stream=None):
    _check(_lib.ppo_test_tc_gemm(mode, _p(A), _p(B), _p(C), M, N, K, _s(stream)))
