"""Developer probe (GPU): fused ABFT-GEMM stage timings under CUDA-graph
replay, FPR on clean data and the D1 scale behind the e_max defaults."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.fused import FusedAbftGemm, plain_gemm  # noqa: E402


def graph_time(fn, iters=50, reps=5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / iters * 1e3)
    return best  # us per call (inputs L2-resident: back-to-back replays)


def main():
    torch.manual_seed(0)
    for (m, k, n) in [(4096, 4096, 4096), (8192, 4096, 11008), (8192, 11008, 4096)]:
        A = torch.randn(m, k, device="cuda").bfloat16()
        B = torch.randn(k, n, device="cuda").bfloat16()
        C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        flops = 2 * m * n * k
        for mode in ("online", "offline"):
            g = FusedAbftGemm(B, mode=mode)
            counts = torch.zeros(5, dtype=torch.int64, device="cuda")
            t = {}
            t["plain"] = graph_time(lambda: plain_gemm(A, B, out=C))
            t["all"] = graph_time(lambda: g(A, out=C, counts=counts))
            t["gemm"] = graph_time(lambda: g(A, out=C, counts=counts, stages=2))
            t["tail"] = graph_time(lambda: g(A, out=C, counts=counts, stages=4))
            counts.zero_()
            r = g(A, out=C, counts=counts)
            torch.cuda.synchronize()
            ratio = (r.diff1.abs() / r.T).max().item()
            s = " ".join(f"{kk}={v:.1f}" for kk, v in t.items())
            print(f"{mode:7s} {m}x{k}x{n}: {s} us | fused {flops/t['all']/1e6:.0f} TFLOP/s plain "
                  f"{flops/t['plain']/1e6:.0f} overhead {100*(t['all']/t['plain']-1):.1f}% | e_max={g.opts.e_max:g} "
                  f"counts={counts.tolist()} max|D1|/T={ratio:.3g}", flush=True)
            g.close()


if __name__ == "__main__":
    main()
