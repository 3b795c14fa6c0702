"""Stage timings of the FP32 / FP64 fused path (CUDA-graph replays, CUDA
events, L2 flushed): GEMM with the ABFT epilogue (stage 2), plain GEMM
(2|8), the A pass with the in-kernel verdicts (4), the whole call (0).
usage: wide_probe.py [n] [passes] [fp64]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.fused import FusedAbftGemm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dt = torch.float64 if (len(sys.argv) > 3 and sys.argv[3] == "fp64") else torch.float32
torch.manual_seed(0)
A = torch.randn(n, n, device="cuda", dtype=dt)
B = torch.randn(n, n, device="cuda", dtype=dt)
g = FusedAbftGemm(B, tf32_passes=passes)
C = torch.empty(n, n, device="cuda", dtype=dt)
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
counts = torch.zeros(6, dtype=torch.int64, device="cuda")
out = {"n": n, "dtype": str(dt), "tf32_passes": passes}
for name, st in (("all", 0), ("gemm_abft_epilogue", 2), ("gemm_plain", 2 | 8), ("a_pass_verdicts", 4)):
    for _ in range(3):
        g(A, out=C, counts=counts, stages=st)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        g(A, out=C, counts=counts, stages=st)
    ts = []
    for i in range(13):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        gr.replay()
        e.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    out[name + "_us"] = round(ts[len(ts) // 2], 1)
print(json.dumps(out))
