"""TF32 and FP64 peaks of this B200 the same way the driver measures the
BF16 one (MEASURED_PEAKS.json: cuBLAS via torch.matmul, 8192^3, best of 10
back-to-back): TF32 tensor cores (allow_tf32), FP64 (cuBLAS DGEMM), plus
the SIMT FP32 GEMM for reference. -> profiles/r02_peaks_tf32_fp64.json"""
import json

import torch

n = 8192
out = {"how": "torch.matmul (cuBLAS) n^3 = 8192^3, 2 n^3 flop, best of 10 back-to-back, CUDA events"}
for name, dt, tf32 in (("tf32_tflops", torch.float32, True), ("fp32_simt_tflops", torch.float32, False),
                       ("fp64_tflops", torch.float64, False), ("bf16_tflops_recheck", torch.bfloat16, False)):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dt)
    b = torch.randn(n, n, device="cuda", dtype=dt)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        a @ b
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    out[name] = 2.0 * n ** 3 / (best * 1e-3) / 1e12
    del a, b
print(json.dumps(out))
