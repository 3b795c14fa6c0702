"""Launch each fused-kernel variant REPS times in a fixed order (dev, GPU) so
that an ncu launch list at locked clocks gives deterministic per-variant
kernel durations:

  ncu --clock-control base --metrics gpu__time_duration.sum --csv \\
      --log-file out.csv python tools/variants_once.py [MxKxN]
  python tools/variants_once.py --parse out.csv

Variants (name, VABFT_DEBUG_STATS, stage mask) as in tools/ablate.py."""
import csv
import os
import statistics
import sys

VARIANTS = [("plain", None, None), ("epi", "3", 2), ("st_nomath", "2", 2), ("st_noload", "1", 2),
            ("gemm+stats", "0", 2), ("arrive_only", "7", 0), ("no_stats_half", "8", 0), ("no_final_half", "9", 0),
            ("full", "0", 0)]
REPS = 5


def run(shape):
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2602_08043_b200.fused import FusedAbftGemm, plain_gemm
    m, k, n = shape
    torch.manual_seed(int(os.environ.get("SEED", "0")))
    A = torch.randn(m, k, device="cuda").bfloat16()
    B = torch.randn(k, n, device="cuda").bfloat16()
    C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    g = FusedAbftGemm(B)
    counts = torch.zeros(6, dtype=torch.int64, device="cuda")
    g(A, out=C, counts=counts)  # first use: workspace identities (not counted: parse skips it)
    for name, dbg, stages in VARIANTS:
        for _ in range(REPS):
            if dbg is None:
                plain_gemm(A, B, out=C)
            else:
                os.environ["VABFT_DEBUG_STATS"] = dbg
                g(A, out=C, counts=counts, stages=stages)
    torch.cuda.synchronize()
    counts.zero_()
    os.environ["VABFT_DEBUG_STATS"] = "0"
    g(A, out=C, counts=counts)
    print("counts [rows, detected, located, nan, slow_stats]:", counts.tolist(), file=sys.stderr)


def parse(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and "tc_gemm" in r[4]
            and r[-3] == "gpu__time_duration.sum"]
    t = [float(r[-1]) / 1000.0 for r in rows][1:]  # drop the warm-up launch
    base = None
    for i, (name, _, _) in enumerate(VARIANTS):
        v = statistics.median(t[i * REPS:(i + 1) * REPS])
        base = base or v
        print(f"{name:12s} {v:8.1f} us  {100 * (v / base - 1):+6.1f}%")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--parse":
        parse(sys.argv[2])
    else:
        run(tuple(int(x) for x in sys.argv[1].split("x")) if len(sys.argv) > 1 else (4096, 4096, 4096))
