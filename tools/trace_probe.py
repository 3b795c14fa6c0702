"""Dev (GPU): per-CTA timeline of one fused launch (VABFT_TRACE=1):
start, MMA end, epilogue end (incl. verification), statistics end, pre-teardown, end."""
import ctypes, os, sys
os.environ["VABFT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch  # noqa: E402
from paper_2602_08043_b200 import _capi  # noqa: E402
from paper_2602_08043_b200.fused import FusedAbftGemm, plain_gemm  # noqa: E402
lib = _capi.lib
lib.vabft_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int, ctypes.c_int]
arg = sys.argv[1] if len(sys.argv) > 1 else "4096"
m, k, n = (int(x) for x in arg.split("x")) if "x" in arg else (int(arg),) * 3
A = torch.randn(m, k, device="cuda").bfloat16(); B = torch.randn(k, n, device="cuda").bfloat16()
if os.environ.get("MIXED"):  # rows outside the exactness guard (bench mixed_scale): 64 rows, half their entries ~1e-10
    rows = torch.arange(0, m, max(1, m // 64), device="cuda")[:64]
    tiny = torch.rand(len(rows), k, device="cuda") < 0.5
    A[rows] = torch.where(tiny, A[rows].float() * 1e-10, A[rows].float()).bfloat16()
g = FusedAbftGemm(B)
plain = bool(os.environ.get("PLAIN"))
Cc = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda") if os.environ.get("FLUSH") else None
dbg = os.environ.get("VABFT_DEBUG_STATS", "0")
for it in range(4):
    buf = (ctypes.c_ulonglong * (148 * 8))()
    lib.vabft_debug_trace(buf, 148 * 8, 1)
    if flush is not None:
        flush.zero_()
    torch.cuda.synchronize()
    res = plain_gemm(A, B, out=Cc, cta_mode=1) if plain else g(A)
    torch.cuda.synchronize()
    lib.vabft_debug_trace(buf, 148 * 8, 0)
t = np.array(buf, dtype=np.int64).reshape(148, 8).astype(np.float64)
t0 = t[:, 0].min()
r = (t - t0) / 1000.0
names = ["start", "mma_end", "epi_end", "stats_end", "pre_teardown", "end"]
print(f"mixed={bool(os.environ.get('MIXED'))} plain={plain} pair={os.environ.get('VABFT_PAIR','1')} debug={dbg} n={m} flush={flush is not None}")
for c, nm in enumerate(names):
    v = r[:, c][t[:, c] > 0]
    if v.size:
        print(f"  {nm:13s} min {v.min():7.1f} med {np.median(v):7.1f} max {v.max():7.1f} us  (n={v.size})")
sh_ns, sh_n = t[:, 6], t[:, 7]
print(f"  stats-half calls: total {int(sh_n.sum())}, max per CTA {int(sh_n.max())}, "
      f"mean duration {sh_ns.sum() / max(sh_n.sum(), 1) / 1000:.2f} us, max CTA total {sh_ns.max() / 1000:.1f} us")
if not plain and res.counts is not None:
    print("  counts [rows, detected, located, nan, slow_stats, corrected]:", res.counts.tolist())
dbg4 = (ctypes.c_ulonglong * 4)()
lib.vabft_debug_tail(dbg4, 1)
print("  tail slow-row paths (last 4 launches): integer exact", dbg4[0], "fallback", dbg4[1])
late = np.argsort(-r[:, 5])[:6]
print("  latest-ending CTAs (cta: mma_end epi_end stats_end pre_teardown end):")
for i in late:
    print("   ", int(i), [round(float(r[i, c]), 1) if t[i, c] > 0 else None for c in (1, 2, 3, 4, 5)])
