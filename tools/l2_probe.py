"""Dev (GPU): is the pair-tile mainloop bound chip-wide (L2 -> SMEM) or per SM?
Runs the plain and fused BF16 kernels with the persistent grid capped at P
pairs (VABFT_MAX_PAIRS, one subprocess per P) on M = 256 * P / 4 x 4096 x K,
i.e. exactly 4 pair tiles per pair (last-wave split off), and prints the time
per pair tile and the per-SM rate. A chip-wide bandwidth bound shows up as
faster tiles when fewer pairs run; a per-SM bound as a flat line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(P, K, raster):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2602_08043_b200.fused import FusedAbftGemm, plain_gemm
    M, N = 256 * P // 4, 4096
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    g = FusedAbftGemm(B)
    out = {"pairs": P, "M": M, "N": N, "K": K}
    for name, fn in (("plain", lambda: plain_gemm(A, B, out=C, cta_mode=1)), ("fused", lambda: g(A, out=C))):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(30):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        ts.sort()
        t = ts[len(ts) // 2]
        out[name + "_us"] = round(t, 1)
        out[name + "_us_per_tile"] = round(t / 4, 2)
        out[name + "_tflops_per_sm"] = round(2 * M * N * K / (t * 1e-6) / 1e12 / (2 * P), 3)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child(int(sys.argv[2]), int(sys.argv[3]), 0)
        sys.exit(0)
    K = int(os.environ.get("K", "4096"))
    for P in (72, 64, 56, 48, 36, 24, 16, 8):
        env = dict(os.environ, VABFT_MAX_PAIRS=str(P), VABFT_SPLIT_LAST="0")
        subprocess.run([sys.executable, __file__, "child", str(P), str(K)], env=env, check=False)
