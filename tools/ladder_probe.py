"""Dev (GPU): overhead ladder of the fused BF16 kernel by ablation
(VABFT_DEBUG_STATS, one subprocess per mode): 1 no statistics loads, 2 no
statistics math, 3 ABFT epilogue only (no statistics warps), 7 no
verification, 8 no statistics half, 9 no final half; 'plain' = ABFT compiled
out. Shapes: MxNxK (default the C2 shape and a 4-tiles-per-pair shape)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(shape, mode):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2602_08043_b200.fused import FusedAbftGemm, plain_gemm
    M, N, K = (int(x) for x in shape.split("x"))
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    if mode == "plain":
        fn = lambda: plain_gemm(A, B, out=C, cta_mode=1)  # noqa: E731
    else:
        g = FusedAbftGemm(B)
        fn = lambda: g(A, out=C)  # noqa: E731
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(40):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    t = ts[len(ts) // 2]
    print(json.dumps({"shape": shape, "mode": mode, "us": round(t, 1), "tflops": round(2 * M * N * K / t / 1e6, 1)}),
          flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "child":
        child(sys.argv[2], sys.argv[3])
        sys.exit(0)
    shapes = [a for a in sys.argv[1:] if "x" in a] or ["4096x4096x4096", "4608x4096x4096"]
    modes = os.environ.get("MODES", "plain,0,1,2,3,7,8,9").split(",")
    rasters = os.environ.get("RASTERS", "").split(",") if os.environ.get("RASTERS") else [None]
    for shape in shapes:
        for raster in rasters:
            for mode in modes:
                env = dict(os.environ)
                if mode != "plain":
                    env["VABFT_DEBUG_STATS"] = mode
                if raster:
                    env["VABFT_RASTER_GROUP"] = raster
                    print("raster", raster, end=" ", flush=True)
                subprocess.run([sys.executable, __file__, "child", shape, mode], env=env, check=False)
