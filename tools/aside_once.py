"""One wide A-side pass (FP32 4096 x 4096) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_08043_b200.fused import FusedAbftGemm
a = torch.randn(4096, 4096, device="cuda"); b = torch.randn(4096, 4096, device="cuda")
g = FusedAbftGemm(b)
g(a, stages=4)
torch.cuda.synchronize()
