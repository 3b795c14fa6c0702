"""Compare the plain tcgen05 GEMM built with 4 vs 3 pipeline stages (dev experiment)."""
import ctypes, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
libs = {"4": os.path.join(ROOT, "paper_2602_08043_b200", "libvabft_b200.so"), "3": os.path.join(ROOT, "tools", "libvabft_stages3.so")}
for (m, n, k) in [(4096, 4096, 4096), (8192, 11008, 4096), (8192, 4096, 11008)]:
    a = torch.randn(m, k, device="cuda").bfloat16(); b = torch.randn(k, n, device="cuda").bfloat16()
    c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for name, path in libs.items():
        lib = ctypes.CDLL(path)
        st = torch.cuda.current_stream().cuda_stream
        f = lambda: lib.vabft_gemm_plain(0, 0, ctypes.c_int64(m), ctypes.c_int64(n), ctypes.c_int64(k), ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(c.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        for _ in range(5): f()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20): f()
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1) / 20 * 1e3)
        print(f"stages={name} {m}x{n}x{k}: {best:.1f} us {2*m*n*k/best/1e6:.0f} TFLOP/s", flush=True)
