"""Multi-rank host logic on CPU (gloo, world_size 2): GEMM-batch plans,
N-slice sharding with slice-local verification, and the counter all-reduce.
The per-slice computation here is the CPU oracle (test infrastructure); on a
GPU box the same slices run through the fused kernel."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_08043_b200.sharding import (allreduce_counts, globalize_location, merge_counts,
                                            plan_gemm_batch, shard_columns, shard_trials)

LLAMA = [(8192, k, n) for k, n in [(4096, 4096)] * 4 + [(4096, 11008)] * 2 + [(11008, 4096)]] * 32


def test_plan_covers_and_balances():
    for world in (1, 2, 4, 8):
        plan = plan_gemm_batch(LLAMA, world)
        flat = sorted(i for r in plan for i in r)
        assert flat == list(range(len(LLAMA)))
        loads = [sum(2 * LLAMA[i][0] * LLAMA[i][1] * LLAMA[i][2] for i in r) for r in plan]
        assert max(loads) / (sum(loads) / world) < 1.02
    assert plan_gemm_batch(LLAMA, 3) == plan_gemm_batch(LLAMA, 3)  # deterministic


def test_shard_columns():
    for n in (8, 96, 768, 4096, 11008):
        for world in (1, 2, 4, 8):
            sl = shard_columns(n, world)
            assert sl[0][0] == 0 and sl[-1][1] == n
            assert all(a % 8 == 0 for a, _ in sl)
            assert all(sl[i][1] == sl[i + 1][0] for i in range(world - 1))


def test_shard_trials_partition():
    for t in (1, 7, 1000, 10**6):
        for w in (1, 2, 3, 8):
            rs = [shard_trials(t, w, r) for r in range(w)]
            assert sum(len(r) for r in rs) == t and rs[0].start == 0 and rs[-1].stop == t


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    P = oracle.port()
    m, k, n = 24, 40, 48
    A, B = P.trial_inputs(m, k, n, "fp32", "uniform:-1,1", 11, 0)
    n0, n1 = shard_columns(n, world)[rank]
    Bs = np.ascontiguousarray(B[:, n0:n1])
    e = P.encode_and_multiply(A, Bs, "fp32", "offline")
    src = e.c.copy()
    # one planted error in a column owned by rank 1, row 5
    planted = (5, 30)
    if n0 <= planted[1] < n1:
        src[planted[0], planted[1] - n0] += 3.0
    T = np.full(m, 1e-3)
    v = P.verify(src, e.row_check1, e.row_check2, T, "fp32", "offline")
    counts = torch.tensor([m, int(v["detected"].sum()), int((v["location"] >= 0).sum()), 0], dtype=torch.int64)
    allreduce_counts(counts)
    locs = [globalize_location(int(x), n0) for x in v["location"]]
    gathered = [None] * world
    dist.all_gather_object(gathered, locs)
    if rank == 0:
        result_q.put((counts.tolist(), gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_nshard_and_counts():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    counts, locs = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert counts[0] == 48  # 24 rows verified on each rank
    assert counts[1] == 1 and counts[2] == 1  # only the owning slice flags row 5
    assert locs[1][5] == 30 and locs[0][5] == -1


def test_merge_counts():
    assert merge_counts([[1, 2, 3, 4], [10, 20, 30, 40]]) == [11, 22, 33, 44]


def test_bench_spawns_ranks_dry_run():
    """bench.py --gpus 2 starts two ranks itself (torch.distributed.run) when
    WORLD_SIZE is unset; --dry-run exercises the plan / slices / counter
    all-reduce over gloo without a GPU."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    for cfg, gemms in (("llama", 112), ("c2", 1), ("nsplit", 1)):
        out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run",
                              "--config", cfg], capture_output=True, text=True, timeout=240, env=env)
        assert out.returncode == 0, out.stderr[-2000:]
        line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
        assert line["n_gpus"] == 2 and line["rank0_gemms"] == gemms
        assert line["all_reduced_gemms"] == (224 if cfg == "llama" else 2)
        if cfg == "nsplit":
            assert line["rank0_columns"] == [0, 5504]
