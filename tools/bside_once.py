"""Run the per-weight B-side pass a few times (for ncu). usage: bside_once.py [dtype K N]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200 import _capi  # noqa: E402
from paper_2602_08043_b200.device import ptr, stream_ptr  # noqa: E402
from paper_2602_08043_b200.fused import FusedAbftGemm  # noqa: E402

dt = getattr(torch, sys.argv[1]) if len(sys.argv) > 1 else torch.bfloat16
k, n = (int(x) for x in (sys.argv[2:4] if len(sys.argv) >= 4 else (4096, 4096)))
torch.manual_seed(0)
B = torch.randn(k, n, device="cuda").to(dt)
g = FusedAbftGemm(B)
for _ in range(3):
    _capi.check(_capi.lib.vabft_bside_update(g.h, ptr(B), stream_ptr()))
torch.cuda.synchronize()
print("ok")
