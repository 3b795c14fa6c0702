"""Developer smoke check of the plain tcgen05 GEMM against torch.matmul (GPU)."""
import ctypes
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2602_08043_b200", "libvabft_b200.so"))
lib.vabft_gemm_plain.restype = ctypes.c_int
lib.vabft_last_error.restype = ctypes.c_char_p


def run(m, n, k, fmt="bf16", kmajor=False, timeit=False):
    dt = torch.bfloat16 if fmt == "bf16" else torch.float16
    torch.manual_seed(0)
    a = torch.randn(m, k, device="cuda").to(dt)
    b = torch.randn(k, n, device="cuda").to(dt)
    bb = b.t().contiguous() if kmajor else b
    c = torch.empty(m, n, device="cuda", dtype=dt)
    f = 0 if fmt == "bf16" else 1
    st = torch.cuda.current_stream().cuda_stream

    def call():
        r = lib.vabft_gemm_plain(f, int(kmajor), ctypes.c_int64(m), ctypes.c_int64(n), ctypes.c_int64(k),
                                 ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(bb.data_ptr()),
                                 ctypes.c_void_p(c.data_ptr()), ctypes.c_void_p(st))
        if r != 0:
            raise RuntimeError(lib.vabft_last_error().decode())

    call()
    torch.cuda.synchronize()
    ref = (a.float() @ b.float())
    err = (c.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    ok = err <= 1e-2 * scale + 1e-3
    msg = f"{fmt} kmajor={kmajor} {m}x{n}x{k}: max|err|={err:.4g} scale={scale:.4g} {'OK' if ok else 'FAIL'}"
    if timeit:
        for _ in range(5):
            call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = 20
        e0.record()
        for _ in range(iters):
            call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        tf = 2 * m * n * k / ms / 1e9
        # torch reference timing
        e0.record()
        for _ in range(iters):
            torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        ms_t = e0.elapsed_time(e1) / iters
        msg += f" | ours {ms*1e3:.1f} us {tf:.0f} TFLOP/s | torch {ms_t*1e3:.1f} us {2*m*n*k/ms_t/1e9:.0f} TFLOP/s"
    print(msg, flush=True)
    return ok


if __name__ == "__main__":
    allok = True
    for (m, n, k) in [(128, 256, 64), (256, 512, 128), (200, 264, 72), (1024, 768, 768)]:
        for km in (False, True):
            allok &= run(m, n, k, "bf16", km)
    allok &= run(512, 512, 512, "fp16", False)
    allok &= run(4096, 4096, 4096, "bf16", False, timeit=True)
    allok &= run(4096, 4096, 4096, "bf16", True, timeit=True)
    allok &= run(8192, 8192, 8192, "bf16", True, timeit=True)
    sys.exit(0 if allok else 1)
