"""Seeded synthetic inputs for the PPO optimizer step (OpenAI Five, arXiv 1912.06680).

This module is shared by the oracle tests, the GPU parity tests and ``bench.py``.
It holds NONE of the method's arithmetic -- no GAE, no LSTM, no loss, no Adam.  It
only draws random numbers shaped like the paper's workload ("Input
recipe") and states the paper's constants.  Random numbers that the method
consumes (e.g. the noise that turns the current log-prob into a behaviour
log-prob) are returned as inputs; each side then does its own arithmetic.

Citations: ``P:n`` = PAPER.md line n (section in brackets).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# Paper constants
# ---------------------------------------------------------------------------

#: Factorised action heads, P:303-368 [App. Action Space, Table target types]:
#: primary (<=30), Delay 4, Unit selection 189, Teleport selection 189,
#: Offset regular / caster / ward 81 each.
HEAD_NAMES = ("primary", "delay", "unit", "teleport",
              "offset_regular", "offset_caster", "offset_ward")
HEAD_SIZES = (30, 4, 189, 189, 81, 81, 81)
N_HEADS = len(HEAD_SIZES)
N_LOGITS = sum(HEAD_SIZES)          # 655
A_OUT = N_LOGITS + 1                # + value, "another linear projection" P:618
N_PRIMARY = HEAD_SIZES[0]

#: Action target types, Table target types P:350-368 -> heads the action reads.
#: Delay is "never ignored"; the primary head is always read.
TARGET_TYPES = {
    "no_target":   ("primary", "delay"),
    "point":       ("primary", "delay", "offset_caster"),
    "unit":        ("primary", "delay", "unit"),
    "unit_offset": ("primary", "delay", "unit", "offset_regular"),
    "teleport":    ("primary", "delay", "teleport", "offset_regular"),
    "ward":        ("primary", "delay", "offset_ward"),
}
TARGET_TYPE_NAMES = tuple(TARGET_TYPES)

#: Hyperparameters, Table hyperparams P:894-933 (Baseline column) and P:1254-1255.
HYPER = dict(
    T_step=4.0 / 30.0,      # frameskip 4 at 30 fps, P:959-961 (paper prints 0.133 s)
    horizon_s=180.0,        # GAE horizon
    lam=0.95,               # GAE lambda
    clip_eps=0.2,           # PPO clipping
    c_v=1.0,                # value loss weight
    c_e=0.01,               # entropy coefficient
    lr=5e-5,                # learning rate
    beta1=0.9,
    beta2=0.999,
    adam_eps=1e-8,          # not printed; reading Q4
    clip_sigma=5.0,         # "+-5 sqrt(v)"
    T=16,                   # LSTM unroll length
    segment=256,            # steps per rollout segment
)


@dataclass(frozen=True)
class Config:
    """Shape of one optimizer step.  B counts LSTM sequences (one hero's 16-step
    window); a paper "sample" is 5 of them."""
    H: int
    D: int
    B: int
    T: int = 16
    head_sizes: tuple = field(default=HEAD_SIZES)
    #: NEXT-4 aux heads (n_win, n_rank, n_bld) appended after the value (DESIGN Q24)
    aux: tuple = field(default=(0, 0, 0))

    @property
    def A(self) -> int:
        return sum(self.head_sizes) + 1 + sum(self.aux)

    @property
    def rows(self) -> int:
        return self.T * self.B


#: configs[0] of BASELINE.json: H=128, obs 256, 32 sequences x 16 steps.
TINY = Config(H=128, D=256, B=32)
#: configs[1]: the paper's 4096-unit LSTM; D=4032 from the parameter budget (DESIGN Q1).
FULL = Config(H=4096, D=4032, B=38400)


# ---------------------------------------------------------------------------
# Helpers (representation only)
# ---------------------------------------------------------------------------

def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (ties to even); returns float32.
    A storage-format conversion, used so both sides see bit-identical inputs."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return (rounded & 0xFFFFFFFF).astype(np.uint32).view(np.float32).reshape(a.shape)


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def target_type_table(seed: int = 1234) -> np.ndarray:
    """Seeded target type (index into TARGET_TYPE_NAMES) for each of the 30 primary
    actions.  Primary 0 is noop (no target)."""
    rng = _rng(seed)
    tt = rng.integers(0, len(TARGET_TYPE_NAMES), size=N_PRIMARY)
    tt[0] = 0
    return tt.astype(np.int32)


def heads_on_table(head_sizes=HEAD_SIZES, seed: int = 1234) -> np.ndarray:
    """[30][n_heads] uint8: which heads the primary action reads."""
    tt = target_type_table(seed)
    tab = np.zeros((N_PRIMARY, len(head_sizes)), np.uint8)
    for p in range(N_PRIMARY):
        for name in TARGET_TYPES[TARGET_TYPE_NAMES[tt[p]]]:
            tab[p, HEAD_NAMES.index(name)] = 1
    return tab


# ---------------------------------------------------------------------------
# Generators
# ---------------------------------------------------------------------------

def make_params(cfg: Config, seed: int, bo_scale: float = 0.0) -> dict:
    """Canonical-layout float32 parameters.  Gate blocks [i; f; g; o] (PyTorch order),
    one LSTM bias (DESIGN Q14).  W_x, W_h, b ~ U(+-1/sqrt(H)); W_o ~ N(0, 0.01^2);
    b_o ~ N(0, bo_scale^2) (0 in the bench recipe)."""
    rng = _rng(seed)
    H, D, A = cfg.H, cfg.D, cfg.A
    s = 1.0 / np.sqrt(H)
    return dict(
        Wx=rng.uniform(-s, s, size=(4 * H, D)).astype(np.float32),
        Wh=rng.uniform(-s, s, size=(4 * H, H)).astype(np.float32),
        b=rng.uniform(-s, s, size=(4 * H,)).astype(np.float32),
        Wo=(0.01 * rng.standard_normal((A, H))).astype(np.float32),
        bo=(bo_scale * rng.standard_normal(A)).astype(np.float32),
    )


def make_sequences(cfg: Config, seed: int, pad_frac: float = 0.0,
                   tt_seed: int = 1234) -> dict:
    """One minibatch of B sequences x T steps, time-major [T][B][.].

    x ~ N(0,1) clipped to (-5,5) (post-normalisation range), rounded to bf16.
    c0 ~ N(0,1); h0 = sigmoid-like bounded draw: h0 = u*w with u~U(0,1), w~U(-1,1)
    (any bounded |h0|<1 state is a valid stored rollout state).
    Availability: noop always, each other primary w.p. 7.1/29 (mean 8.1).
    Actions: uniform over available primaries; parameter heads uniform.
    logp_noise ~ N(0, 0.1^2): behaviour log-prob = current log-prob + noise.
    """
    rng = _rng(seed)
    T, B, H, D = cfg.T, cfg.B, cfg.H, cfg.D
    x = np.clip(rng.standard_normal((T, B, D), dtype=np.float32), -5.0, 5.0)
    x = round_bf16(x)
    c0 = rng.standard_normal((B, H)).astype(np.float32)
    h0 = (rng.uniform(0, 1, (B, H)) * rng.uniform(-1, 1, (B, H))).astype(np.float32)

    avail = (rng.uniform(0, 1, (T, B, N_PRIMARY)) < 7.1 / 29.0).astype(np.uint8)
    avail[..., 0] = 1
    # primary: uniform over available entries
    u = rng.uniform(0, 1, (T, B, N_PRIMARY)) * avail
    primary = np.argmax(u, axis=-1).astype(np.int32)
    act = np.zeros((T, B, len(cfg.head_sizes)), np.int32)
    act[..., 0] = primary
    for k, n in enumerate(cfg.head_sizes[1:], start=1):
        act[..., k] = rng.integers(0, n, size=(T, B))
    head_on = heads_on_table(cfg.head_sizes, tt_seed)[primary]
    valid = np.ones((T, B), np.uint8)
    if pad_frac > 0:
        # pad the tail of some sequences (episode ended inside the window)
        npad = rng.integers(1, T + 1, size=B)
        padded = rng.uniform(0, 1, B) < pad_frac
        for b in np.nonzero(padded)[0]:
            valid[T - npad[b]:, b] = 0
    logp_noise = (0.1 * rng.standard_normal((T, B))).astype(np.float32)
    return dict(x=x, h0=h0, c0=c0, act=act, head_on=head_on.astype(np.uint8),
                avail=avail, valid=valid, logp_noise=logp_noise)


def make_rollouts(R: int, L: int, seed: int, p_done: float = 1.0 / 20000) -> dict:
    """R rollout streams of L steps: r ~ N(0,1) (post-normalisation),
    V ~ N(0,1) with the bootstrap V[L], done ~ Bernoulli(p_done) (~20k steps per
    game)."""
    rng = _rng(seed)
    r = rng.standard_normal((R, L)).astype(np.float32)
    V = rng.standard_normal((R, L + 1)).astype(np.float32)
    d = (rng.uniform(0, 1, (R, L)) < p_done).astype(np.uint8)
    return dict(r=r, V=V, done=d)


#: NEXT-4 defaults: win probability, net-worth rank among the 5 heroes, the enemy team's 18
#: buildings (11 towers, 6 barracks, the ancient) (DESIGN Q24).
AUX_SIZES = (1, 5, 18)


def make_aux(R: int, L: int, aux: tuple, seed: int, p_last: float = 0.1,
             p_event: float = 1.0 / 2000) -> dict:
    """Per 256-step segment: whether it is the game's last (p_last), the outcome (win 0/1)
    and final net-worth rank (0-based), building events [R][L][n_bld] (Bernoulli p_event per
    step), and the model's bootstrap predictions after the last step: win ~ U(0,1), rank a
    normalised U(0,1) vector, buildings ~ U(0, 0.3)."""
    n_win, n_rank, n_bld = aux
    rng = _rng(seed)
    boot = [rng.uniform(0, 1, size=(R, n_win))]
    rk = rng.uniform(0, 1, size=(R, n_rank))
    boot.append(rk / np.maximum(rk.sum(axis=1, keepdims=True), 1e-12) if n_rank else rk)
    boot.append(rng.uniform(0, 0.3, size=(R, n_bld)))
    return dict(last=(rng.random(R) < p_last).astype(np.uint8),
                outcome=(rng.random(R) < 0.5).astype(np.float32),
                rank=rng.integers(0, max(n_rank, 1), size=R).astype(np.int32),
                events=(rng.random((R, L, n_bld)) < p_event).astype(np.uint8),
                boot=np.concatenate(boot, axis=1).astype(np.float32))


def make_logits(rows: int, A: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """Head outputs for isolated loss tests: N(0, scale^2) float32 [rows][A]."""
    return (scale * _rng(seed).standard_normal((rows, A))).astype(np.float32)


# ---------------------------------------------------------------------------
# Device-side generation for large B (bench / full-size sampled parity).  Same recipe,
# torch Philox generator on the device; still no method arithmetic.
# ---------------------------------------------------------------------------

def torch_sequences(cfg: Config, seed: int, device, x_dtype=None, tt_seed: int = 1234) -> dict:
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    T, B, H, D = cfg.T, cfg.B, cfg.H, cfg.D
    x_dtype = x_dtype or torch.bfloat16
    x = torch.empty((T, B, D), dtype=x_dtype, device=device)
    for t in range(T):  # chunked to bound the fp32 temporary
        x[t] = torch.randn((B, D), generator=g, device=device).clamp_(-5.0, 5.0).to(x_dtype)
    c0 = torch.randn((B, H), generator=g, device=device)
    h0 = torch.rand((B, H), generator=g, device=device) * (torch.rand((B, H), generator=g, device=device) * 2 - 1)
    avail = (torch.rand((T, B, N_PRIMARY), generator=g, device=device) < 7.1 / 29.0).to(torch.uint8)
    avail[..., 0] = 1
    u = torch.rand((T, B, N_PRIMARY), generator=g, device=device) * avail
    primary = torch.argmax(u, dim=-1).to(torch.int32)
    act = torch.empty((T, B, len(cfg.head_sizes)), dtype=torch.int32, device=device)
    act[..., 0] = primary
    for k, n in enumerate(cfg.head_sizes[1:], start=1):
        act[..., k] = torch.randint(0, n, (T, B), generator=g, device=device, dtype=torch.int32)
    tab = torch.from_numpy(heads_on_table(cfg.head_sizes, tt_seed)).to(device)
    head_on = tab[primary.long()]
    logp_noise = 0.1 * torch.randn((T, B), generator=g, device=device)
    return dict(x=x, h0=h0, c0=c0, act=act, head_on=head_on, avail=avail,
                logp_noise=logp_noise)


def torch_rollouts(R: int, L: int, seed: int, device, p_done: float = 1.0 / 20000) -> dict:
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed + 7)
    return dict(rew=torch.randn((R, L), generator=g, device=device),
                val=torch.randn((R, L + 1), generator=g, device=device),
                done=(torch.rand((R, L), generator=g, device=device) < p_done).to(torch.uint8))


def torch_aux(R: int, L: int, aux: tuple, seed: int, device, p_last: float = 0.1,
              p_event: float = 1.0 / 2000) -> dict:
    """Device twin of make_aux (same recipe, torch Philox draws)."""
    import torch
    n_win, n_rank, n_bld = aux
    g = torch.Generator(device=device)
    g.manual_seed(seed + 11)
    rk = torch.rand((R, n_rank), generator=g, device=device)
    rk = rk / rk.sum(dim=1, keepdim=True).clamp_min(1e-12)
    boot = torch.cat([torch.rand((R, n_win), generator=g, device=device), rk,
                      0.3 * torch.rand((R, n_bld), generator=g, device=device)], dim=1)
    return dict(last=(torch.rand(R, generator=g, device=device) < p_last).to(torch.uint8),
                outcome=(torch.rand(R, generator=g, device=device) < 0.5).float(),
                rank=torch.randint(0, max(n_rank, 1), (R,), generator=g, device=device,
                                   dtype=torch.int32),
                events=(torch.rand((R, L, n_bld), generator=g, device=device) < p_event)
                .to(torch.uint8),
                boot=boot.contiguous())


def torch_params(cfg: Config, seed: int, device, bo_scale: float = 0.0) -> dict:
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed + 13)
    H, D, A = cfg.H, cfg.D, cfg.A
    s = 1.0 / float(np.sqrt(H))
    def U(*shape):
        return (torch.rand(shape, generator=g, device=device) * 2 - 1) * s
    return dict(Wx=U(4 * H, D), Wh=U(4 * H, H), b=U(4 * H),
                Wo=0.01 * torch.randn((A, H), generator=g, device=device),
                bo=bo_scale * torch.randn((A,), generator=g, device=device))
