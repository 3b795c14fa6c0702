"""Clock / power under each fused-kernel variant (dev, GPU): long CUDA-graph
replays while an NVML thread samples the SM clock and board power."""
import os
import statistics
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.fused import FusedAbftGemm, plain_gemm  # noqa: E402


def run(fn, iters, h):
    for _ in range(3):
        fn()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(50):
            fn()
    torch.cuda.synchronize()
    clk, pw, stop = [], [], [False]

    def sampler():
        while not stop[0]:
            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
            time.sleep(0.005)

    g.replay()
    torch.cuda.synchronize()
    th = threading.Thread(target=sampler)
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters // 50):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    stop[0] = True
    th.join()
    n = len(clk)
    tail = slice(n // 3, None)  # steady state
    return e0.elapsed_time(e1) / iters * 1e3, statistics.median(clk[tail]), statistics.median(pw[tail])


def main():
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    torch.manual_seed(0)
    m = k = n = 4096
    A = torch.randn(m, k, device="cuda").bfloat16()
    B = torch.randn(k, n, device="cuda").bfloat16()
    C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    g = FusedAbftGemm(B)
    counts = torch.zeros(5, dtype=torch.int64, device="cuda")
    variants = [("plain", None, None), ("epi", "3", 2), ("st_nomath", "2", 2), ("st_noload", "1", 2),
                ("gemm+stats", "0", 2), ("arrive_only", "7", 0), ("full", "0", 0)]
    for rep in range(2):
        for name, dbg, stages in variants:
            if dbg is None:
                fn = lambda: plain_gemm(A, B, out=C)  # noqa: E731
            else:
                os.environ["VABFT_DEBUG_STATS"] = dbg
                g(A, out=C, counts=counts)
                fn = lambda: g(A, out=C, counts=counts, stages=stages)  # noqa: E731
            us, mhz, watts = run(fn, 3000, h)
            print(f"rep{rep} {name:11s} {us:7.1f} us  sm {mhz:5.0f} MHz  {watts:6.0f} W  "
                  f"{2 * m * n * k / us / 1e6:6.0f} TFLOP/s  {2 * m * n * k / us / 1e6 / mhz * 1000:6.1f} TF/s/GHz",
                  flush=True)
    os.environ["VABFT_DEBUG_STATS"] = "0"


if __name__ == "__main__":
    main()
