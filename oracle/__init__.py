"""ORACLE -- test infrastructure only.

A plain, slow, obviously-correct float64 NumPy implementation of the PPO optimizer
step of OpenAI Five (arXiv 1912.06680, §3.2).  It exists to
check the CUDA path, and nothing in the product path may import it: only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs use it.  It shares no code with
``paper_1912_06680_b200`` (no kernels, headers, helpers, tables or constants);
the only shared module is ``synth`` (seeded input draws, no method arithmetic).

Every function follows the paper's equations in the paper's order, in canonical
layout (gate blocks [i; f; g; o], separate W_x, W_h, b, W_o, b_o), with no
blocking, fusion or reordering.  Readings of silent/ambiguous passages are the
DESIGN.md table (Q1-Q16).  Pins live in tests/test_oracle_*.py.

Parity status ("Oracle pins"):
  gae            pinned (closed forms, brute force, SPEC worked example, printed gamma)
  lstm fwd/bwd   pinned (zero-param closed form, torch.nn.LSTM fp64, finite differences)
  heads + loss   pinned (clip/entropy closed forms, masking invariants, finite differences)
  adam + clip    pinned (textbook Adam via torch.optim.Adam, hand-evaluated steps, clip window)
  dp average     pinned (shard identity)
  buffer         sampler pinned to splitmix64's published test vector; gather = indexing
  step           composition of the above, pinned end-to-end by finite differences
  aux (NEXT-4)   labels = the paper's piecewise equation + closed-form 2-min discount; losses:
                 ln 2 / ln n closed forms, finite differences; routing: FD of the composed
                 step (trunk sees L_ppo + w c_win L_win, aux rows the whole loss)
  lstm_input_grad (NEXT-4) = torch autograd's x.grad
  infer (NEXT-3) state carry = 2-step LSTM; Gumbel-max frequencies = softmax (chi-square);
                 masks, target-type table, logp = the loss oracle's log pi
"""
from .gae import gamma_from_horizon, gae, segments_to_sequences  # noqa: F401
from .lstm import lstm_forward, lstm_backward, lstm_input_grad  # noqa: F401
from .loss import heads_forward, heads_backward, ppo_loss, STAT_NAMES  # noqa: F401
from .adam import adam_clip  # noqa: F401
from .step import ppo_step, dp_average  # noqa: F401
from . import buffer  # noqa: F401
from . import infer  # noqa: F401
from . import aux  # noqa: F401
