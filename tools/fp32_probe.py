"""FP32 fused V-ABFT GEMM (tcgen05 3xTF32 / 1xTF32) throughput vs the plain
kernel and cuBLAS (FP32 SIMT and TF32)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_08043_b200.fused import plain_gemm, FusedAbftGemm


def t(fn, it=10):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it


for n in (2048, 4096, 8192):
    a = torch.randn(n, n, device='cuda'); b = torch.randn(n, n, device='cuda')
    fl = 2 * n**3
    torch.backends.cuda.matmul.allow_tf32 = False
    tc = t(lambda: a @ b)
    torch.backends.cuda.matmul.allow_tf32 = True
    tt = t(lambda: a @ b)
    g3 = FusedAbftGemm(b, mode="online"); g1 = FusedAbftGemm(b, mode="online", tf32_passes=1, e_max=2e-3)
    tf3 = t(lambda: g3(a)); tf1 = t(lambda: g1(a))
    tp = t(lambda: plain_gemm(a, b))
    print(json.dumps({"n": n, "cublas_fp32_tf": fl / tc / 1e9, "cublas_tf32_tf": fl / tt / 1e9,
                      "plain_3xtf32_incl_splits_tf": fl / tp / 1e9, "fused_3xtf32_tf": fl / tf3 / 1e9,
                      "fused_1xtf32_tf": fl / tf1 / 1e9}))
