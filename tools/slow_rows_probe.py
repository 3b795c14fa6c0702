"""1xTF32 / 3xTF32 fused 4096^3 over many seeds: sequential-fallback (tie)
row count vs device time per call (CUDA graph replay, L2 flushed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_08043_b200.fused import FusedAbftGemm
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
passes = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for seed in range(int(sys.argv[2]) if len(sys.argv) > 2 else 16):
    torch.manual_seed(seed)
    a = torch.randn(4096, 4096, device="cuda"); b = torch.randn(4096, 4096, device="cuda")
    g = FusedAbftGemm(b, tf32_passes=passes)
    c = torch.zeros(6, dtype=torch.int64, device="cuda")
    for _ in range(3):
        g(a, counts=c)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        g(a, counts=c)
    c.zero_()
    ts = []
    for _ in range(5):
        flush.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); gr.replay(); e.record(); torch.cuda.synchronize()
        ts.append(round(s.elapsed_time(e) * 1e3, 1))
    print(passes, seed, "slow_rows/call", c[4].item() // 5, "us", min(ts), flush=True)
    g.close()
