"""Counters of wide-format fused calls (slow-stats rows etc.), several seeds,
with per-call device time (CUDA graph replay, L2 flushed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_08043_b200.fused import FusedAbftGemm
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for dt, passes in ((torch.float32, 1), (torch.float32, 3), (torch.float64, 3)):
    for seed in range(3):
        torch.manual_seed(seed)
        a = torch.randn(4096, 4096, device="cuda", dtype=dt); b = torch.randn(4096, 4096, device="cuda", dtype=dt)
        g = FusedAbftGemm(b, tf32_passes=passes)
        c = torch.zeros(6, dtype=torch.int64, device="cuda")
        for _ in range(3):
            g(a, counts=c)
        torch.cuda.synchronize()
        c.zero_()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            g(a, counts=c)
        ts = []
        for _ in range(5):
            flush.zero_()
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            s.record(); gr.replay(); e.record(); torch.cuda.synchronize()
            ts.append(round(s.elapsed_time(e) * 1e3, 1))
        print(dt, passes, seed, c.tolist(), ts, flush=True)
        g.close()
