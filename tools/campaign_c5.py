"""C5: fault-injection campaign over GPT-2-small / ViT-B/16 shaped GEMMs
(SURVEY §8(d) C5): FP32-accumulator bits 0-31 (online) and BF16 output bits
0-15 (offline), Set0To1, >= 1e6 trials in total, detection and location
rates per (shape, bit). M trials per fused launch (DeviceCampaign); on N
ranks each rank runs its share of launches with its own seed and the
counters are all-reduced over NCCL (the path's only collective).

  python tools/campaign_c5.py [--trials-per-bit 8192] > profiles/r01_campaign_c5.jsonl
  python -m torch.distributed.run --nproc-per-node 8 tools/campaign_c5.py ...
"""
import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_08043_b200.campaign import DeviceCampaign  # noqa: E402
from paper_2602_08043_b200.emax import default_e_max  # noqa: E402

SHAPES = {  # (M, K, N): GPT-2 small with M = 1024 tokens, ViT-B/16 with M = 32 x 197
    "gpt2.qkv": (1024, 768, 2304), "gpt2.proj": (1024, 768, 768), "gpt2.fc": (1024, 768, 3072),
    "gpt2.fc2": (1024, 3072, 768),
    "vitb.qkv": (6304, 768, 2304), "vitb.proj": (6304, 768, 768), "vitb.fc": (6304, 768, 3072),
    "vitb.fc2": (6304, 3072, 768),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials-per-bit", type=int, default=8192)
    ap.add_argument("--shapes", default=",".join(SHAPES))
    ap.add_argument("--dist", default="normal:1e-6,1")
    ap.add_argument("--b-trials-per-bit", type=int, default=256, help="B-operand trials (one per launch)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    total = 0
    t_all = time.time()
    for name in args.shapes.split(","):
        m, k, n = SHAPES[name]
        # (mode, fault target, bits, trials per bit): FP32-accumulator bits
        # online, output bits offline, BF16 A / B operand bits (online verify)
        plan = (("online", "output", range(32), args.trials_per_bit),
                ("offline", "output", range(16), args.trials_per_bit),
                ("online", "A", range(16), args.trials_per_bit),
                ("online", "B", range(16), args.b_trials_per_bit))
        for mode, target, bits, tpb in plan:
            e_max = default_e_max("bf16", mode, k)
            camp = DeviceCampaign(m, k, n, dist=args.dist, mode=mode, e_max=e_max, seed=1000 * rank + 7)
            for b in bits:
                per_rank = (tpb + world - 1) // world
                t0 = time.time()
                o = camp.run(b, per_rank, reduce=world > 1, target=target)  # all-reduced counters
                total += o.trials
                if rank == 0:
                    print(json.dumps({"shape": name, "mkn": [m, k, n], "mode": mode, "target": target, "bit": b,
                                      "e_max": e_max, "ranks": world, **o.as_dict(),
                                      "seconds": round(time.time() - t0, 3)}), flush=True)
            camp.close()
    if rank == 0:
        print(json.dumps({"summary": True, "trials_total": total if world == 1 else None,
                          "seconds": round(time.time() - t_all, 1), "ranks": world}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
