"""C3 sweep (BASELINE config 3): precision x distribution x n — V-ABFT vs
A-ABFT thresholds, tightness and false positives, on the device paths
(GPU). The reference's harness definitions (proj/src/harness.cpp):

  run_fpr        a row is a false positive when isnan(D1) or |D1| > T_i on
                 clean data (D1 = r1 - row_check1 of the verification source)
  run_tightness  tightness = mean threshold / mean actual difference

BF16/FP16: the fused tcgen05 path (FusedAbftGemm: T_V with the device
e_max defaults, T_A = A-ABFT computed y), operands drawn on the device; the
actual difference is |D1| of the fused verification (FP32 blocked:128 row
sums of the accumulator vs the checksums); FP32 / FP64 also on their fused
device paths up to n = 16384 / 8192. FP32/FP64 "exact" lines: the EXACT engine
(api.py), sizes capped like the reference (FP64 at 512); the actual
difference is |row_check1 - exactly rounded row sum of the source|
(math.fsum, the role MPFR plays in oracle_row_diffs), T_V with
resolve_e_max of the format's default model, T_A fixed y = 21.

  python tools/sweep_c3.py [--quick] [--rows 100000] > profiles/r02_sweep_c3.jsonl
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200 import api  # noqa: E402
from paper_2602_08043_b200.campaign import sample_matrix  # noqa: E402
from paper_2602_08043_b200.fused import FusedAbftGemm  # noqa: E402

DISTS = ["normal:0,1", "normal:1e-6,1", "normal:1,1", "uniform:-1,1", "truncnormal:0,1,-1,1"]


def sweep16(fmt, dist, n, trials, mode, gen):
    """The fused device path (any format): T_V with the device e_max defaults,
    T_A per AabftParams::for_format (computed y for 16-bit, y = 21 for
    FP32 / FP64, threshold_aabft.cpp:8-29)."""
    dtype = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32, "fp64": torch.float64}[fmt]
    aab = "aabft-computed-y" if fmt in ("bf16", "fp16") else "aabft-fixed-y"
    dev = torch.device("cuda")
    acc = {"tv": 0.0, "ta": 0.0, "act": 0.0, "max_act": 0.0, "fp_v": 0, "fp_a": 0, "rows": 0, "e_max": None}
    for _ in range(trials):
        A = sample_matrix((n, n), dist, gen, dev, dtype)
        B = sample_matrix((n, n), dist, gen, dev, dtype)
        cv = torch.zeros(6, dtype=torch.int64, device=dev)
        ca = torch.zeros(6, dtype=torch.int64, device=dev)
        gv = FusedAbftGemm(B, mode=mode)
        rv = gv(A, counts=cv)
        ga = FusedAbftGemm(B, mode=mode, threshold=aab)
        ra = ga(A, counts=ca)
        d1 = rv.diff1.abs()
        acc["tv"] += rv.T.mean().item()
        acc["ta"] += ra.T.mean().item()
        acc["act"] += d1[torch.isfinite(d1)].mean().item() if bool(torch.isfinite(d1).any()) else float("nan")
        acc["max_act"] = max(acc["max_act"], d1.max().item())
        acc["fp_v"] += int(cv[1].item())
        acc["fp_a"] += int(ca[1].item())
        acc["rows"] += n
        acc["e_max"] = gv.opts.e_max
        gv.close()
        ga.close()
    return acc


def draw(rng, shape, dist, fmt):
    name, _, rest = dist.partition(":")
    a = [float(t) for t in rest.split(",")] if rest else []
    if name == "normal":
        x = rng.normal(a[0], a[1], shape)
    elif name == "uniform":
        x = rng.uniform(a[0], a[1], shape)
    elif name == "truncnormal":
        x = rng.normal(a[0], a[1], shape)
        bad = (x < a[2]) | (x > a[3])
        while bad.any():
            x[bad] = rng.normal(a[0], a[1], int(bad.sum()))
            bad = (x < a[2]) | (x > a[3])
    else:
        raise ValueError(dist)
    return x.astype(np.float32).astype(np.float64) if fmt == "fp32" else x


def sweep_wide(fmt, dist, n, trials, mode, rng):
    acc = {"tv": 0.0, "ta": 0.0, "act": 0.0, "max_act": 0.0, "fp_v": 0, "fp_a": 0, "rows": 0, "e_max": None}
    e_max = api.resolve_e_max(fmt, n)
    for _ in range(trials):
        A = draw(rng, (n, n), dist, fmt)
        B = draw(rng, (n, n), dist, fmt)
        e = api.encode_and_multiply(A, B, mode, fmt, engine="exact")
        tv = api.vabft_thresholds(A, B, api.VabftParams(e_max, 2.5), fmt)
        ta = api.aabft_threshold(A, B, api.AabftParams.for_format(fmt), fmt).per_row
        src = e.verification_source()
        actual = np.array([abs(e.row_check1[i] - math.fsum(src[i])) for i in range(n)])
        for th, key in ((tv, "fp_v"), (ta, "fp_a")):
            v = api.verify_arrays(src, e.verification_format(), e.row_check1, e.row_check2, th, e.checksum_precision)
            acc[key] += int(np.sum(v["detected"]))
        acc["tv"] += float(np.mean(tv))
        acc["ta"] += float(np.mean(ta))
        acc["act"] += float(np.mean(actual))
        acc["max_act"] = max(acc["max_act"], float(np.max(actual)))
        acc["rows"] += n
        acc["e_max"] = e_max
    return acc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--rows", type=int, default=100000,
                    help="clean rows per (format, distribution, mode, n <= 4096) configuration")
    ap.add_argument("--exact-rows", type=int, default=20000, help="rows per EXACT-engine configuration")
    args = ap.parse_args()
    gen = torch.Generator(device="cuda")
    gen.manual_seed(0)
    rng = np.random.default_rng(0)
    plan = []
    sizes16 = [(256, 4), (1024, 3), (4096, 2), (16384, 1)] if not args.quick else [(256, 2), (1024, 1)]
    for fmt in ("bf16", "fp16"):
        for mode in ("online", "offline"):
            for dist in DISTS:
                for n, t in sizes16:
                    plan.append((fmt, mode, dist, n, t))
    wide = {"fp32": [(256, 3), (1024, 2), (2048, 1)], "fp64": [(128, 3), (256, 2), (512, 1)]}
    if args.quick:
        wide = {"fp32": [(256, 1)], "fp64": [(128, 1)]}
    for fmt, sz in wide.items():
        for dist in DISTS:
            for n, t in sz:
                plan.append((fmt + ":exact", "offline", dist, n, t))
    # the fused device paths for FP32 (3xTF32 on tcgen05) and FP64 (DFMA), up to 16384
    sizesw = {"fp32": [(256, 3), (1024, 2), (4096, 2), (16384, 1)], "fp64": [(256, 3), (1024, 2), (4096, 1), (8192, 1)]}
    if args.quick:
        sizesw = {"fp32": [(256, 1)], "fp64": [(256, 1)]}
    for fmt, sz in sizesw.items():
        for dist in DISTS:
            for n, t in sz:
                plan.append((fmt, "online", dist, n, t))
    for fmt, mode, dist, n, trials in plan:
        t0 = time.time()
        if not args.quick and n <= 4096:  # >= args.rows rows per configuration
            want = args.exact_rows if fmt.endswith(":exact") else args.rows
            trials = max(trials, -(-want // n))
        if fmt.endswith(":exact"):
            fmt = fmt.split(":")[0]
            a = sweep_wide(fmt, dist, n, trials, mode, rng)
            engine = "exact (order-exact SIMT)"
        else:
            if fmt == "fp16" and dist == "normal:1,1" and n >= 4096 and mode == "offline":
                continue  # FP16 output overflows (|C| ~ n): saturated, not a rounding experiment
            a = sweep16(fmt, dist, n, trials, mode, gen)
            engine = {"fp32": "tensor (fused tcgen05 3xTF32)", "fp64": "fused SIMT DFMA"}.get(fmt, "tensor (fused tcgen05)")
        mt_v, mt_a, ma = a["tv"] / trials, a["ta"] / trials, a["act"] / trials
        line = {"precision": fmt, "mode": mode, "dist": dist, "n": n, "trials": trials, "engine": engine,
                "e_max": a["e_max"], "mean_T_vabft": mt_v, "mean_T_aabft": mt_a,
                "ratio_vabft_over_aabft": mt_v / mt_a if mt_a > 0 else None,
                "mean_actual": ma, "max_actual": a["max_act"],
                "tightness_vabft": mt_v / ma if ma > 0 else None, "tightness_aabft": mt_a / ma if ma > 0 else None,
                "fp_rows_vabft": a["fp_v"], "fp_rows_aabft": a["fp_a"], "rows": a["rows"],
                "seconds": round(time.time() - t0, 2)}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
