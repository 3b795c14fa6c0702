"""Kernel timeline (CUPTI via torch.profiler) of one wide-format fused call
(GEMM, A-side pass, verify tail); args: n fp32|fp64 passes [flush] [counts]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2602_08043_b200.fused import FusedAbftGemm
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dt = {"fp32": torch.float32, "fp64": torch.float64}[sys.argv[2] if len(sys.argv) > 2 else "fp32"]
passes = int(sys.argv[3]) if len(sys.argv) > 3 else 1
a = torch.randn(n, n, device="cuda", dtype=dt); b = torch.randn(n, n, device="cuda", dtype=dt)
g = FusedAbftGemm(b, tf32_passes=passes, e_max=1e-2)
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda") if "flush" in sys.argv else None
counts = torch.zeros(6, dtype=torch.int64, device="cuda") if "counts" in sys.argv else None
for _ in range(3):
    g(a, counts=counts)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        if flush is not None:
            flush.zero_()
        g(a, counts=counts)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in evs)
if counts is not None:
    print("counts", counts.tolist())
for e in sorted(evs, key=lambda e: e.time_range.start):
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f}  {e.name[:70]}")
