"""Run the fwd-shape test GEMM once per (variant, grid policy) for ncu DRAM comparisons."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1912_06680_b200 import _lib as L  # noqa: E402

M, N, K = 38400, 16384, 8192
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn((M, K), generator=g, device="cuda").bfloat16()
B = torch.randn((N, K), generator=g, device="cuda").bfloat16()
C = torch.empty((M, N), device="cuda")
for mode in (0, 8):
    for allt in ("0", "1"):
        os.environ["PPO_GRID_ALL_TILES"] = allt
        L.test_tc_gemm(mode, A, B, C, M, N, K)
torch.mm(A, B.t())
torch.cuda.synchronize()
print("ok")
