"""Developer probe (GPU): fused ABFT-GEMM timing, FPR on clean data, D1 scale
for e_max calibration, injection sanity."""
import sys
import os
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.fused import FusedAbftGemm, plain_gemm  # noqa: E402


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3  # us


def main():
    torch.manual_seed(0)
    for (m, k, n) in [(4096, 4096, 4096), (8192, 4096, 11008)]:
        A = torch.randn(m, k, device="cuda").bfloat16()
        B = torch.randn(k, n, device="cuda").bfloat16()
        for mode in ("online", "offline"):
            g = FusedAbftGemm(B, mode=mode, e_max=1.0)
            counts = torch.zeros(4, dtype=torch.int64, device="cuda")
            r = g(A, counts=counts)
            torch.cuda.synchronize()
            rel = (r.diff1.abs() / 1.0).max().item()
            # |D1| relative to |checksum| proxy: sum_j |C_ij|
            denom = r.C.float().abs().sum(1).double()
            ratio = (r.diff1.abs() / denom).max().item()
            us_f = timeit(lambda: g(A, out=r.C, verdicts=True, counts=counts))
            us_p = timeit(lambda: plain_gemm(A, B, out=r.C))
            tf = 2 * m * n * k / us_f / 1e6
            print(f"{mode:7s} {m}x{k}x{n}: fused {us_f:.1f} us ({tf:.0f} TFLOP/s) plain {us_p:.1f} us "
                  f"({2*m*n*k/us_p/1e6:.0f}) overhead {100*(us_f/us_p-1):.1f}% | max|D1|={rel:.3g} "
                  f"max|D1|/sum|C|={ratio:.3g} T(e=1) mean={r.T.mean().item():.3g}", flush=True)
            # FPR at the default e_max
            g2 = FusedAbftGemm(B, mode=mode)
            c2 = torch.zeros(4, dtype=torch.int64, device="cuda")
            r2 = g2(A, counts=c2)
            torch.cuda.synchronize()
            print(f"   default e_max={g2.opts.e_max:g}: counts={c2.tolist()} max|D1|/T={(r2.diff1.abs()/r2.T).max().item():.3g}",
                  flush=True)
            g.close()
            g2.close()


if __name__ == "__main__":
    main()
