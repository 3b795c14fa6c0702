"""Run one fused stage a few times (for ncu --set full captures).
usage: stage_once.py M K N STAGES [mode]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.fused import FusedAbftGemm  # noqa: E402

m, k, n, stages = (int(x) for x in sys.argv[1:5])
mode = sys.argv[5] if len(sys.argv) > 5 else "online"
torch.manual_seed(0)
A = torch.randn(m, k, device="cuda").bfloat16()
B = torch.randn(k, n, device="cuda").bfloat16()
g = FusedAbftGemm(B, mode=mode)
counts = torch.zeros(5, dtype=torch.int64, device="cuda")
for _ in range(2):
    g(A, counts=counts)            # full path first: valid workspace partials
for _ in range(3):
    g(A, counts=counts, stages=stages)
torch.cuda.synchronize()
print("ok", counts.tolist())
