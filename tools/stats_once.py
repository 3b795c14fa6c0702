"""Launches for the statistics-pass ncu summary (profiles/r02_ncu_stats_passes.json):
per-weight B-side pass BF16 / FP32 (4096^2) and the FP32 fused call's A pass + combine
(4096^3, 1xTF32), two of each, L2 flushed before every launch."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.fused import FusedAbftGemm  # noqa: E402

torch.manual_seed(0)
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for dt in (torch.bfloat16, torch.float32):
    B = torch.randn(4096, 4096, device="cuda").to(dt)
    g = FusedAbftGemm(B, tf32_passes=1) if dt == torch.float32 else FusedAbftGemm(B)
    for _ in range(2):
        flush.zero_()
        g.update_weight(B)
    if dt == torch.float32:
        A = torch.randn(4096, 4096, device="cuda")
        for _ in range(2):
            flush.zero_()
            g(A)
    torch.cuda.synchronize()
    g.close()
print("ok")
