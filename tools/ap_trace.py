"""A-pass timeline (VABFT_APART_TRACE=1 prints %globaltimer stamps per launch):
standalone (stages=4) and inside the full FP32 call. usage: ap_trace.py [n] [passes]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.fused import FusedAbftGemm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 1
torch.manual_seed(0)
A = torch.randn(n, n, device="cuda")
B = torch.randn(n, n, device="cuda")
g = FusedAbftGemm(B, tf32_passes=passes)
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for st in (4, 4, 0, 0):
    flush.zero_()
    print(f"stages={st}", file=sys.stderr, flush=True)
    g(A, stages=st)
    torch.cuda.synchronize()
