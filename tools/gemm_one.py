"""One GEMM of a given shape through cuBLAS (torch.mm) and through the tcgen05 variants
(single CTA, CTA pair), for ncu side-by-side captures.   python tools/gemm_one.py wgrad"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1912_06680_b200 import _lib as L  # noqa: E402

SHAPES = {"fwd": (38400, 16384, 8192, False, False), "wgrad": (16384, 8192, 76800, True, True),
          "bwd": (38400, 4096, 16384, False, True), "square": (8192, 8192, 8192, False, False)}
M, N, K, a_mn, b_mn = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "fwd"]
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn((K, M) if a_mn else (M, K), generator=g, device="cuda").bfloat16()
B = torch.randn((K, N) if b_mn else (N, K), generator=g, device="cuda").bfloat16()
C = torch.empty((M, N), device="cuda")
mode = (1 if b_mn else 0) | (2 if a_mn else 0)
Am = A.t() if a_mn else A
Bm = B if b_mn else B.t()
torch.mm(Am, Bm)
L.test_tc_gemm(mode, A, B, C, M, N, K)
L.test_tc_gemm(mode | 8, A, B, C, M, N, K)
if a_mn and b_mn:
    L.test_tc_gemm(mode | 8 | 16, A, B, C, M, N, K)
torch.cuda.synchronize()
print("ok")
