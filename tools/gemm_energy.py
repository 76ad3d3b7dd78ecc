"""Energy and throughput of the tcgen05 GEMM variants vs cuBLAS (torch.mm) on the step's GEMM
shapes, measured with the NVML energy counter while each runs back-to-back for ~3 s.

    python tools/gemm_energy.py
The step is power-capped (1 kW), so TFLOP per joule decides throughput."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_1912_06680_b200 import _lib as L  # noqa: E402

pynvml.nvmlInit()
dev = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())


def measure(fn, flop, seconds=3.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    clocks = []
    stop = [False]

    def sampler():
        while not stop[0]:
            clocks.append(pynvml.nvmlDeviceGetClockInfo(dev, pynvml.NVML_CLOCK_SM))
            time.sleep(0.05)

    th = threading.Thread(target=sampler, daemon=True)
    e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(dev)
    t0 = time.perf_counter()
    th.start()
    n = 0
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    while time.perf_counter() - t0 < seconds:
        for _ in range(4):
            fn()
        n += 4
        torch.cuda.synchronize()
    s1.record()
    torch.cuda.synchronize()
    e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(dev)
    stop[0] = True
    ms = s0.elapsed_time(s1)
    joules = (e1 - e0) / 1e3
    clocks.sort()
    return dict(tflops=flop * n / (ms / 1e3) / 1e12, watts=joules / (ms / 1e3),
                tflop_per_j=flop * n / joules / 1e12, mhz=clocks[len(clocks) // 2] if clocks else 0,
                ms=ms / n)


def run(name, M, N, K, a_mn, b_mn):
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn((K, M) if a_mn else (M, K), generator=g, device="cuda").bfloat16()
    B = torch.randn((K, N) if b_mn else (N, K), generator=g, device="cuda").bfloat16()
    C = torch.empty((M, N), device="cuda")
    flop = 2.0 * M * N * K
    mode = (1 if b_mn else 0) | (2 if a_mn else 0)
    Am = A.t() if a_mn else A
    Bm = B if b_mn else B.t()
    res = {}
    res["cublas"] = measure(lambda: torch.mm(Am, Bm, out=C.bfloat16()) if False else torch.mm(Am, Bm), flop)
    res["tc_1cta"] = measure(lambda: L.test_tc_gemm(mode, A, B, C, M, N, K), flop)
    res["tc_pair"] = measure(lambda: L.test_tc_gemm(mode | 8, A, B, C, M, N, K), flop)
    for k, v in res.items():
        print(f"{name:10s} {k:8s} {v['tflops']:7.1f} TF/s  {v['watts']:6.0f} W  "
              f"{v['tflop_per_j']:5.3f} TFLOP/J  sm {v['mhz']:5.0f} MHz  {v['ms']:8.3f} ms", flush=True)
    del A, B, C
    torch.cuda.empty_cache()


SHAPES = {"square": (8192, 8192, 8192, False, False), "fwd": (38400, 16384, 8192, False, False),
          "wgrad": (16384, 8192, 76800, True, True), "bwd": (38400, 4096, 16384, False, True)}


def sweep(name, rasters, seconds=2.0):
    """tcgen05 variants x rasterisations (PPO_RASTER_TEST) on one shape, plus cuBLAS"""
    M, N, K, a_mn, b_mn = SHAPES[name]
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn((K, M) if a_mn else (M, K), generator=g, device="cuda").bfloat16()
    B = torch.randn((K, N) if b_mn else (N, K), generator=g, device="cuda").bfloat16()
    C = torch.empty((M, N), device="cuda")
    flop = 2.0 * M * N * K
    mode = (1 if b_mn else 0) | (2 if a_mn else 0)
    Am = A.t() if a_mn else A
    Bm = B if b_mn else B.t()
    rows = [("cublas", "-", measure(lambda: torch.mm(Am, Bm), flop, seconds))]
    for r in rasters:
        os.environ["PPO_RASTER_TEST"] = r
        rows.append(("tc_1cta", r, measure(lambda: L.test_tc_gemm(mode, A, B, C, M, N, K), flop, seconds)))
        rows.append(("tc_pair", r, measure(lambda: L.test_tc_gemm(mode | 8, A, B, C, M, N, K), flop, seconds)))
        if a_mn and b_mn:
            rows.append(("tc_pair2", r, measure(lambda: L.test_tc_gemm(mode | 24, A, B, C, M, N, K), flop, seconds)))
    for k, r, v in rows:
        print(f"{name:7s} {k:8s} {r:4s} {v['tflops']:7.1f} TF/s  {v['watts']:6.0f} W  "
              f"{v['tflop_per_j']:5.3f} TFLOP/J  sm {v['mhz']:5.0f} MHz  {v['ms']:8.3f} ms", flush=True)
    del A, B, C
    torch.cuda.empty_cache()


if __name__ == "__main__":
    which = sys.argv[1:] or ["fwd"]
    for nm in which:
        sweep(nm, os.environ.get("RASTERS", "m8,m16,n8,n16,n32").split(","))
