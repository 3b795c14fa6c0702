"""Threshold tightness table (PAPER.md:478-526 protocol, harness run_tightness)
on the device EXACT engine with the reference's Philox trials: full-row
V-ABFT, block-wise V-ABFT (tiles 1024 x 256) and A-ABFT.

  python tools/tightness_table.py [trials multiplier] > profiles/r02_tightness.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.harness import ExperimentConfig, run_tightness  # noqa: E402

SCALE = int(sys.argv[1]) if len(sys.argv) > 1 else 1  # trials multiplier
PLAN = [("fp32", 128, 10), ("fp32", 512, 5), ("fp32", 2048, 2), ("fp64", 128, 10), ("fp64", 512, 3),
        ("bf16", 128, 10), ("bf16", 512, 5), ("bf16", 2048, 2)]
PLAN = [(f, n, t * SCALE) for (f, n, t) in PLAN]
for fmt, n, trials in PLAN:
    methods = ["vabft", "vabft-blockwise", "aabft-fixed-y" if fmt in ("fp32", "fp64") else "aabft-computed-y"]
    cfg = ExperimentConfig(precision=fmt, dist="normal:0,1", m=n, k=n, n=n, trials=trials, seed=0,
                           methods=methods, tile_k=1024, tile_n=256)
    doc = run_tightness(cfg)
    print(json.dumps({"precision": fmt, "n": n, "trials": trials, "e_max": doc["config"]["e_max"],
                      "mean_actual": doc["actual"]["mean"],
                      **{m: {"tightness": doc["methods"][m]["tightness"],
                             "rows_not_covered": doc["methods"][m]["rows_not_covered"]} for m in methods},
                      "seconds": round(doc["wall_time_s"], 2)}), flush=True)
