"""Stats-warp ablation timing (dev): run with VABFT_DEBUG_STATS=0/1/2."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.fused import FusedAbftGemm, plain_gemm  # noqa: E402
from tools.fused_probe import graph_time  # noqa: E402
torch.manual_seed(0)
for (m, k, n) in [(4096, 4096, 4096), (8192, 11008, 4096)]:
    A = torch.randn(m, k, device="cuda").bfloat16(); B = torch.randn(k, n, device="cuda").bfloat16()
    C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    g = FusedAbftGemm(B)
    counts = torch.zeros(5, dtype=torch.int64, device="cuda")
    tp = graph_time(lambda: plain_gemm(A, B, out=C))
    tg = graph_time(lambda: g(A, out=C, counts=counts, stages=2))
    print(f"debug={os.environ.get('VABFT_DEBUG_STATS','0')} {m}x{k}x{n}: plain {tp:.1f} gemm+stats {tg:.1f} (+{100*(tg/tp-1):.1f}%)", flush=True)
