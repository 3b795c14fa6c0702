"""Counters of one wide-format fused call (slow-stats rows etc.)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_08043_b200.fused import FusedAbftGemm
for dt, passes in ((torch.float32, 1), (torch.float32, 3), (torch.float64, 3)):
    a = torch.randn(4096, 4096, device="cuda", dtype=dt); b = torch.randn(4096, 4096, device="cuda", dtype=dt)
    g = FusedAbftGemm(b, tf32_passes=passes)
    c = torch.zeros(6, dtype=torch.int64, device="cuda")
    g(a, counts=c)
    torch.cuda.synchronize()
    print(dt, passes, c.tolist())
