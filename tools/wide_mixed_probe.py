"""FP32 fused call on mixed-scale activations (64 rows with half their entries
~1e-10): time vs clean (CUDA graph replays, L2 flushed) and the slow-stats
count (rows whose exact sum needed the sequential fallback)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.fused import FusedAbftGemm  # noqa: E402

n = 4096
torch.manual_seed(0)
A = torch.randn(n, n, device="cuda")
B = torch.randn(n, n, device="cuda")
Am = A.clone()
rows = torch.arange(0, n, n // 64, device="cuda")[:64]
tiny = torch.rand(len(rows), n, device="cuda") < 0.5
Am[rows] = torch.where(tiny, Am[rows] * 1e-10, Am[rows])
g = FusedAbftGemm(B, tf32_passes=1)
C = torch.empty(n, n, device="cuda")
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
out = {}
for name, X in (("clean", A), ("mixed", Am)):
    counts = torch.zeros(6, dtype=torch.int64, device="cuda")
    for _ in range(2):
        g(X, out=C, counts=counts)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g(X, out=C, counts=counts)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    counts.zero_()
    g(X, out=C, counts=counts)
    torch.cuda.synchronize()
    out[name] = {"us": sorted(ts)[3], "counts": counts.tolist()}
print(json.dumps(out))
