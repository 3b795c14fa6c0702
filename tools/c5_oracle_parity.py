"""C5 per-trial parity against the reference.

For every GPT-2-small / ViT-B/16 layer shape and every bit
of the campaign plan — FP32-accumulator bits 0-31 verified online, BF16
output bits 0-15 verified offline, Set0To1 — one fused launch runs M trials
(one planned fault per row, injected in the tcgen05 epilogue). A sample of
the launch's trials is re-verified by the reference compiled from its own
sources (oracle/_ref): thresholds vabft_thresholds(A[S], B), the row
checksums (the reference's row_sums composition in the fused path's FP32
NativeBlocked(128) checksum precision) and verify() on the device's own
post-injection accumulator / output. Per trial the applicability, the
verdict and the located column must agree bit for bit; the line per
(shape, mode, bit) records the counts and the agreement.

  python tools/c5_oracle_parity.py [--sample 96] [--fmt bf16|fp16|fp32|fp64] [--shapes ...]
"""
import argparse
import json
import os
import sys
import time
import zlib
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (test infrastructure: the checker)
from paper_2602_08043_b200.campaign import sample_matrix  # noqa: E402
from paper_2602_08043_b200.fused import FusedAbftGemm  # noqa: E402

SHAPES = {
    "gpt2.qkv": (1024, 768, 2304), "gpt2.proj": (1024, 768, 768), "gpt2.fc": (1024, 768, 3072),
    "gpt2.fc2": (1024, 3072, 768),
    "vitb.qkv": (6304, 768, 2304), "vitb.proj": (6304, 768, 768), "vitb.fc": (6304, 768, 3072),
    "vitb.fc2": (6304, 3072, 768),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sample", type=int, default=96, help="trials per launch re-verified by the reference")
    ap.add_argument("--shapes", default=",".join(SHAPES))
    ap.add_argument("--dist", default="normal:1e-6,1")
    ap.add_argument("--fmt", default="bf16", choices=["bf16", "fp16", "fp32", "fp64"],
                    help="operand format: 16-bit — FP32-accumulator bits online, output bits offline; "
                         "FP32 / FP64 — the bits of C (the accumulator), online")
    args = ap.parse_args()
    fmt = args.fmt
    dt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32, "fp64": torch.float64}[fmt]
    sixteen = fmt in ("bf16", "fp16")
    R = oracle.ref() if oracle.have_ref() else oracle.port()
    dev = torch.device("cuda", 0)
    pool = ThreadPoolExecutor(max_workers=os.cpu_count() or 4)
    grand = {"trials": 0, "compared": 0, "agree": 0}
    for name in args.shapes.split(","):
        m, k, n = SHAPES[name]
        gen = torch.Generator(device=dev).manual_seed(zlib.crc32(name.encode()))
        A = sample_matrix((m, k), args.dist, gen, dev, dtype=dt)
        B = sample_matrix((k, n), args.dist, gen, dev, dtype=dt)
        B_h = B.double().cpu().numpy()
        rng = np.random.default_rng(len(name) * 7919 + m)
        plan = ((("online", range(32)), ("offline", range(16))) if sixteen else
                (("online", range(32 if fmt == "fp32" else 64)),))
        for mode, bits in plan:
            g = FusedAbftGemm(B, mode=mode)
            S = np.sort(rng.choice(m, size=min(args.sample, m), replace=False))
            Sd = torch.from_numpy(S).to(dev)
            A_s = A[Sd].double().cpu().numpy()
            # reference thresholds / checksums of the sampled rows, once per (shape, mode):
            # row slices are exact sub-problems; chunks run in parallel
            chunks = np.array_split(np.arange(len(S)), min(len(S), os.cpu_count() or 4))
            th = list(pool.map(lambda c: R.vabft_thresholds(A_s[c], B_h, g.opts.e_max, fmt=fmt)[0], chunks))
            cs = list(pool.map(lambda c: R.blocked_row_checksums(A_s[c], B_h, fmt, mode), chunks))
            T_ref = np.concatenate(th)
            rc1 = np.concatenate([c[0] for c in cs])
            rc2 = np.concatenate([c[1] for c in cs])
            acc = torch.empty(m, n, dtype=torch.float32, device=dev) if (sixteen and mode == "online") else None
            rec = torch.empty(m * 24, dtype=torch.uint8, device=dev)
            for bit in bits:
                t0 = time.time()
                col = torch.randint(0, n, (m,), generator=gen, device=dev, dtype=torch.int32)
                f = {"col": col, "bit": torch.full((m,), bit, dtype=torch.int32, device=dev),
                     "dir": torch.full((m,), 1, dtype=torch.int32, device=dev), "records": rec}
                counts = torch.zeros(6, dtype=torch.int64, device=dev)
                r = g(A, faults=f, counts=counts, accum_out=acc)
                torch.cuda.synchronize()
                applied = rec.view(m, 24)[:, 16:20].contiguous().view(torch.int32).view(m).cpu().numpy() != 0
                src = (acc[Sd] if acc is not None else r.C[Sd]).double().cpu().numpy()
                if sixteen:
                    v = R.verify(src, rc1, rc2, T_ref, "fp32", "offline", accum=(2, 128))
                else:  # C is the accumulator; checksum precision = the format, blocked:128
                    v = R.verify(src, rc1, rc2, T_ref, fmt, "online", accum=(2, 128))
                det = r.detected[Sd].cpu().numpy().astype(bool)
                loc = r.location[Sd].cpu().numpy()
                T_dev = r.T[Sd].cpu().numpy()
                agree = (det == v["detected"]) & (loc == v["location"])
                same_T = np.array_equal(T_dev.view(np.uint64), T_ref.view(np.uint64))
                cols = col[Sd].cpu().numpy()
                app = applied[S]
                line = {"shape": name, "mkn": [m, k, n], "mode": mode, "bit": bit,
                        "fmt": fmt,
                        "target": (("fp32_accumulator" if mode == "online" else fmt + "_output") if sixteen
                                   else fmt + "_C"),
                        "device_trials": m, "device_applicable": int(applied.sum()),
                        "device_detected": int(counts[1].item()),
                        "compared": int(len(S)), "applicable_compared": int(app.sum()),
                        "agree": int(agree.sum()), "thresholds_bit_exact": bool(same_T),
                        "detected_compared": int(v["detected"][app].sum()),
                        "located_correctly_compared": int(((v["location"] == cols) & v["detected"])[app].sum()),
                        "false_positives_unapplicable": int(det[~app].sum()),
                        "s": round(time.time() - t0, 3)}
                grand["trials"] += m
                grand["compared"] += len(S)
                grand["agree"] += int(agree.sum())
                print(json.dumps(line), flush=True)
            g.close()
    print(json.dumps({"summary": grand, "fmt": fmt, "reference": R.name}), flush=True)


if __name__ == "__main__":
    main()
