"""paper_1912_06680_b200 -- a B200-native (sm_100a) PPO optimizer step for the OpenAI Five
4096-unit LSTM policy/value network (arXiv 1912.06680, §3.2).

The product is libppo5.so (C ABI in include/ppo5.h); this package is its thin binding
(`_lib`) and the step composition (`step.PPOOptimizer`).  Importing fails loudly if the
library is not built: there is no CPU fallback.
"""
from . import _lib  # noqa: F401  (raises ImportError if libppo5.so is missing)
from .step import DEFAULT_HYPER, HEAD_SIZES, PPOOptimizer  # noqa: F401

__all__ = ["PPOOptimizer", "HEAD_SIZES", "DEFAULT_HYPER", "_lib"]
