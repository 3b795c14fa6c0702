"""Dev (GPU): fused and plain tcgen05 GEMM, 1-CTA vs CTA-pair kernels, at the
bench shapes (run as: VABFT_PAIR=0|1 python tools/mode_sweep.py), L2 flushed
before each launch, CUDA-graph replay."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.fused import FusedAbftGemm, plain_gemm  # noqa: E402
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
def timed(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    es = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    tot = 0.0
    for a, b in es:
        flush.zero_(); a.record(); fn(); b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in es)
    return ts[len(ts) // 2]
for (m, k, n) in [(4096, 4096, 4096), (8192, 4096, 4096), (8192, 4096, 11008), (8192, 11008, 4096), (8192, 8192, 8192)]:
    A = torch.randn(m, k, device="cuda").bfloat16(); B = torch.randn(k, n, device="cuda").bfloat16()
    C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    g = FusedAbftGemm(B)
    tf = timed(lambda: g(A, out=C)); tp = timed(lambda: plain_gemm(A, B, out=C))
    f = 2 * m * n * k
    print(f"pair={os.environ.get('VABFT_PAIR')} {m}x{k}x{n}: fused {tf:.1f} us {f/tf/1e6:.0f} TF/s | plain {tp:.1f} us {f/tp/1e6:.0f} TF/s | overhead {100*(tf/tp-1):.1f}%", flush=True)
    g.close()
