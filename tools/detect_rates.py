"""Detection / localization rate per bit (BASELINE config 5 protocol at the
reference's campaign shape) — the B200 device campaign beside the
reference's own CPU injection_campaign, same e_max, same fault model
(Set0To1 at a uniform eligible position, faults.hpp:60-62).

Device: DeviceCampaign, M trials per fused launch (campaign.py). Reference:
oracle/_ref injection_campaign (multithreaded), fewer trials. The two draw
different operands (torch vs Philox streams), so the comparison is of
rates; per-trial verdict parity is tests/test_gpu_campaign.py.

  python tools/detect_rates.py [--ref-trials 400] > profiles/r01_detect_rates.jsonl
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_08043_b200.campaign import DeviceCampaign  # noqa: E402
from paper_2602_08043_b200.emax import default_e_max  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=8192)
    ap.add_argument("--ref-trials", type=int, default=400)
    ap.add_argument("--m", type=int, default=128)
    ap.add_argument("--k", type=int, default=1024)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--dist", default="normal:1e-6,1")
    ap.add_argument("--bits-online", default="0-31")
    ap.add_argument("--bits-offline", default="0-15")
    args = ap.parse_args()
    ref = None
    try:
        import oracle
        if oracle.have_ref():
            ref = oracle.ref()
    except Exception:
        ref = None

    def bits(spec):
        lo, _, hi = spec.partition("-")
        return list(range(int(lo), int(hi or lo) + 1))

    for mode, blist in (("offline", bits(args.bits_offline)), ("online", bits(args.bits_online))):
        e_max = default_e_max("bf16", mode, args.k)
        camp = DeviceCampaign(args.m, args.k, args.n, dist=args.dist, mode=mode, e_max=e_max, seed=11,
                              refresh=1)
        for b in blist:
            t0 = time.time()
            o = camp.run(b, args.trials, reduce=False)
            dt = time.time() - t0
            line = {"shape": [args.m, args.k, args.n], "precision": "bf16", "dist": args.dist, "mode": mode,
                    "target": "FP32 accumulator" if mode == "online" else "BF16 output", "bit": b,
                    "e_max": e_max, "device": o.as_dict(), "device_seconds": round(dt, 3)}
            if ref is not None and args.ref_trials > 0:
                t0 = time.time()
                r = ref.injection_campaign(args.m, args.k, args.n, "bf16", args.dist, b, args.ref_trials, 5, mode,
                                           0, e_max)
                line["reference"] = {"trials": int(r[0]), "applicable": int(r[1]), "detected": int(r[2]),
                                     "located_correctly": int(r[3]), "nonfinite_after": int(r[4]),
                                     "detection_rate": (r[2] / r[1]) if r[1] else None,
                                     "localization_accuracy": (r[3] / r[2]) if r[2] else None}
                line["reference_seconds"] = round(time.time() - t0, 3)
                line["reference_cores"] = os.cpu_count()
            print(json.dumps(line), flush=True)
        camp.close()


if __name__ == "__main__":
    main()
