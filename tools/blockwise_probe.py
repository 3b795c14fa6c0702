"""Block-wise V-ABFT on the fused path (BlockwiseFusedGemm) vs the full-row
fused call, 4096^3 BF16 online, the paper's tiles (K-tile 1024, N-block 256):
CUDA-event times (L2 flushed), the device block-wise threshold kernels alone.
usage: blockwise_probe.py [n]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200 import blockwise  # noqa: E402
from paper_2602_08043_b200.fused import FusedAbftGemm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
torch.manual_seed(0)
A = torch.randn(n, n, device="cuda").bfloat16()
B = torch.randn(n, n, device="cuda").bfloat16()
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
bw = blockwise.BlockwiseFusedGemm(B, "bf16", "online", 1024, 256)
full = FusedAbftGemm(B)
C = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
counts = torch.zeros(6, dtype=torch.int64, device="cuda")


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


t_thr = timeit(lambda: blockwise.blockwise_thresholds_device(A, B, "bf16", 1024, 256, bw.e_max))
t_bw = timeit(lambda: bw(A, out=C, counts=counts))
t_full = timeit(lambda: full(A, out=C, counts=counts))
counts.zero_()
r = bw(A, out=C, counts=counts)
torch.cuda.synchronize()
fl = 2.0 * n ** 3
print(json.dumps({"n": n, "tiles": [1024, 256], "blockwise_thresholds_us": t_thr, "blockwise_call_us": t_bw,
                  "blockwise_tflops": fl / t_bw / 1e6, "full_row_fused_us": t_full, "full_row_tflops": fl / t_full / 1e6,
                  "blocks": len(bw.blocks), "rows_flagged": int(r.detected.sum().item()),
                  "counts": counts.tolist()}))
