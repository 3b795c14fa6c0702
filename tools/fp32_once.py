"""One FP32 fused call (3xTF32 and 1xTF32) at 4096^3, for the ncu launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_08043_b200.fused import FusedAbftGemm
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
a = torch.randn(n, n, device="cuda"); b = torch.randn(n, n, device="cuda")
g3 = FusedAbftGemm(b); g1 = FusedAbftGemm(b, tf32_passes=1, e_max=2e-3)
torch.cuda.synchronize()
for _ in range(2):
    g3(a); g1(a)
torch.cuda.synchronize()
