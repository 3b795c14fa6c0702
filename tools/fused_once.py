"""Run the fused V-ABFT GEMM a few times at one shape (for ncu launch lists)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.fused import FusedAbftGemm, plain_gemm  # noqa: E402

m, k, n = (int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else (4096, 4096, 4096)))
mode = sys.argv[4] if len(sys.argv) >= 5 else "online"
torch.manual_seed(0)
A = torch.randn(m, k, device="cuda").bfloat16()
B = torch.randn(k, n, device="cuda").bfloat16()
g = FusedAbftGemm(B, mode=mode)
counts = torch.zeros(6, dtype=torch.int64, device="cuda")
for _ in range(3):
    r = g(A, counts=counts)
    plain_gemm(A, B, out=r.C)
torch.cuda.synchronize()
print("counts", counts.tolist())
