"""Fused-kernel ablation ladder (dev, GPU). For each shape, under CUDA-graph
replay (L2-warm, back-to-back):
  plain        tcgen05 GEMM, ABFT compiled out
  epi          ABFT epilogue only (row partials), no statistics warps
  st_noload    + statistics warps, producer skips the A reloads (math on stale smem)
  st_nomath    + statistics loads, no statistics math
  gemm+stats   GEMM + epilogue + statistics, no verify tail
  full         the product path (in-kernel verify tail)
  tail         the standalone verify tail kernel alone
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.fused import FusedAbftGemm, plain_gemm  # noqa: E402
from tools.fused_probe import graph_time  # noqa: E402

SHAPES = [(4096, 4096, 4096), (8192, 4096, 11008), (8192, 11008, 4096)]


def main():
    torch.manual_seed(0)
    shapes = SHAPES if len(sys.argv) < 2 else [tuple(int(x) for x in s.split("x")) for s in sys.argv[1:]]
    for (m, k, n) in shapes:
        A = torch.randn(m, k, device="cuda").bfloat16()
        B = torch.randn(k, n, device="cuda").bfloat16()
        C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        g = FusedAbftGemm(B)
        counts = torch.zeros(5, dtype=torch.int64, device="cuda")
        t = {"plain": graph_time(lambda: plain_gemm(A, B, out=C))}
        for name, dbg, stages in (("epi", "3", 2), ("st_noload", "1", 2), ("st_nomath", "2", 2),
                                  ("gemm+stats", "0", 2), ("full", "0", 0), ("tail", "0", 4)):
            os.environ["VABFT_DEBUG_STATS"] = dbg
            g(A, out=C, counts=counts)  # first use: workspace identities
            t[name] = graph_time(lambda: g(A, out=C, counts=counts, stages=stages))
        os.environ["VABFT_DEBUG_STATS"] = "0"
        g.close()
        base = t["plain"]
        s = " ".join(f"{kk}={v:.1f}({100 * (v / base - 1):+.1f}%)" for kk, v in t.items())
        print(f"{m}x{k}x{n}: {s}", flush=True)


if __name__ == "__main__":
    main()
