"""Dev (GPU): plain tcgen05 GEMM timing at a few shapes (run with VABFT_PAIR=0/1)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.fused import plain_gemm  # noqa: E402
from tools.fused_probe import graph_time  # noqa: E402
for (m, k, n) in [(18944, 4096, 256), (18944, 16384, 256), (9472, 16384, 512), (4096, 4096, 4096), (8192, 8192, 8192)]:
    A = torch.randn(m, k, device="cuda").bfloat16(); B = torch.randn(k, n, device="cuda").bfloat16()
    C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    t = graph_time(lambda: plain_gemm(A, B, out=C), iters=20, reps=3)
    print(os.environ.get("VABFT_PAIR"), m, k, n, f"{t:.1f} us {2*m*n*k/t/1e6:.0f} TFLOP/s", flush=True)
