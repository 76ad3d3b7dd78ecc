"""Phase trace of one CTA-pair GEMM launch (experiments build with -DPPO_TRACE):
    PPO_NVCC_EXTRA=-DPPO_TRACE python paper_1912_06680_b200/build.py && python tools/trace_gemm.py
Per CTA: cycles from kernel entry to 1 setup done (cluster_sync), 2 first tile fetched,
4 first stage landed (MMA), 5 first tile's last MMA committed, 6 accumulator ready (epilogue),
7 epilogue done, 8 exit, 9 TMEM freed; plus each CTA's entry time (globaltimer) vs the first."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_1912_06680_b200 import _lib as L  # noqa: E402

lib = L._lib
lib.ppo_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for (M, N, K, mode) in [(128, 256, 64, 8), (32, 512, 448, 8), (256, 256, 4096, 8),
                        (600, 16384, 8192, 8), (256, 4096, 64, 8)]:
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda")
    for _ in range(3):
        L.test_tc_gemm(mode, A, B, C, M, N, K)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        L.test_tc_gemm(mode, A, B, C, M, N, K)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    lib.ppo_trace_clear()
    L.test_tc_gemm(mode, A, B, C, M, N, K)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (512 * 32))()
    lib.ppo_trace_read(buf, 512 * 32)
    mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    ntiles = -(-M // 256) * -(-N // 256)
    nct = 2 * min(ntiles, 74)
    t0s = [buf[32 * b] for b in range(nct)]
    tmin = min(t for t in t0s if t)
    print(f"M={M} N={N} K={K} tiles={ntiles}: {us:.1f} us/launch (events, back to back), sm {mhz} MHz")
    for b in range(min(nct, 6)):
        ph = [buf[32 * b + i] for i in range(1, 10)]
        print(f"  cta {b:3d} entry +{(t0s[b] - tmin) / 1e3:7.2f} us  phases(us): " +
              " ".join(f"{i}:{p / mhz:7.2f}" for i, p in zip(range(1, 10), ph) if p))
