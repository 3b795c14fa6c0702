"""One FP64 GEMM of each kind at 4096^3 (for ncu): the DFMA kernel, then cuBLAS."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_08043_b200.fused import plain_gemm
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
a = torch.randn(n, n, device="cuda", dtype=torch.float64)
b = torch.randn(n, n, device="cuda", dtype=torch.float64)
plain_gemm(a, b)
torch.cuda.synchronize()
c = a @ b
torch.cuda.synchronize()
