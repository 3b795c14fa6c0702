"""Small launches of this session's new kernels for compute-sanitizer
(memcheck / racecheck): wide A pass + combine (FP32, FP64, ragged M/K/N),
B-side pass (BF16 with guard-failing rows, FP32 with the fused split),
block-wise thresholds, the 16-bit integer exact-sum path."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200 import blockwise  # noqa: E402
from paper_2602_08043_b200.fused import FusedAbftGemm  # noqa: E402

torch.manual_seed(0)
for dt, (m, k, n) in ((torch.float32, (200, 392, 264)), (torch.float64, (130, 264, 136)), (torch.float32, (64, 128, 64))):
    A = torch.randn(m, k, device="cuda", dtype=dt)
    B = torch.randn(k, n, device="cuda", dtype=dt)
    g = FusedAbftGemm(B, tf32_passes=1) if dt == torch.float32 else FusedAbftGemm(B)
    counts = torch.zeros(6, dtype=torch.int64, device="cuda")
    r = g(A, counts=counts)
    torch.cuda.synchronize()
    assert int(counts[1].item()) == 0, counts.tolist()
    g.close()
A = torch.randn(160, 1024, device="cuda")
rows = torch.arange(0, 160, 7, device="cuda")
A[rows] = torch.where(torch.rand(len(rows), 1024, device="cuda") < 0.5, A[rows] * 1e-10, A[rows])
A = A.bfloat16()
B = torch.randn(1024, 512, device="cuda").bfloat16()
B[::5] = (B[::5].float() * torch.where(torch.rand(B[::5].shape, device="cuda") < 0.3, 1e-9, 1.0)).bfloat16()
g = FusedAbftGemm(B)
counts = torch.zeros(6, dtype=torch.int64, device="cuda")
g(A, counts=counts)
torch.cuda.synchronize()
assert int(counts[4].item()) > 0 and int(counts[1].item()) == 0, counts.tolist()
g.close()
T = blockwise.blockwise_thresholds_device(A, B, "bf16", 384, 128)
bw = blockwise.BlockwiseFusedGemm(B, "bf16", "online", 512, 256, graphs=False)
v = bw(A)
torch.cuda.synchronize()
bw.close()
print("sanitize ok")
