"""Time the per-weight B-side pass (vabft_bside_update: bside_kernel [+ FP32
TF32 split]) as a CUDA-graph replay with CUDA events, L2 flushed between launches.
usage: bside_probe.py [K N] -> one JSON line per format"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200 import _capi  # noqa: E402
from paper_2602_08043_b200.device import ptr, stream_ptr  # noqa: E402
from paper_2602_08043_b200.fused import FusedAbftGemm  # noqa: E402

k, n = (int(x) for x in (sys.argv[1:3] if len(sys.argv) >= 3 else (4096, 4096)))
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for dt in (torch.bfloat16, torch.float16, torch.float32, torch.float64):
    torch.manual_seed(0)
    B = torch.randn(k, n, device="cuda").to(dt)
    g = FusedAbftGemm(B)
    for _ in range(3):
        _capi.check(_capi.lib.vabft_bside_update(g.h, ptr(B), stream_ptr()))
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()  # device time only (no host launch gaps inside the events)
    with torch.cuda.graph(gr):
        _capi.check(_capi.lib.vabft_bside_update(g.h, ptr(B), stream_ptr()))
    ts = []
    for i in range(23):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        gr.replay()
        e.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    byts = B.numel() * B.element_size()
    print(json.dumps({"format": str(dt).split(".")[-1], "K": k, "N": n, "us_median": ts[len(ts) // 2], "us_min": ts[0],
                      "bytes_B": byts, "GBps_median": byts / (ts[len(ts) // 2] * 1e-6) / 1e9}), flush=True)
    g.close()
