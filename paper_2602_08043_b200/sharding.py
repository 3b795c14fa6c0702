"""Multi-GPU partitioning of the V-ABFT path.

The path shards with no operand exchange:
  * batches of independent GEMMs (e.g. the 224 LLaMA-7B layer GEMMs, or
    campaign trials) are partitioned across ranks by a greedy
    longest-processing-time plan on FLOPs;
  * one large GEMM can be split along N: rank g owns the columns
    [n0_g, n1_g) of B and C and verifies that slice as an independent ABFT
    unit (thresholds with n = N_g from slice-local B statistics; a located
    column is slice-local and is shifted by n0_g).
The only collective is the int64 fault-counter all-reduce (sum).
"""
from __future__ import annotations

import heapq
from typing import Iterable, List, Sequence, Tuple


def plan_gemm_batch(shapes: Sequence[Tuple[int, int, int]], world: int) -> List[List[int]]:
    """Greedy LPT assignment of GEMMs (m, k, n) to `world` ranks by 2mkn FLOPs.
    Deterministic: ties broken by index; returns per-rank index lists in
    original order."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(shapes)), key=lambda i: (-2 * shapes[i][0] * shapes[i][1] * shapes[i][2], i))
    heap = [(0, r) for r in range(world)]
    out: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        m, k, n = shapes[i]
        out[r].append(i)
        heapq.heappush(heap, (load + 2 * m * k * n, r))
    return [sorted(v) for v in out]


def shard_columns(n: int, world: int, align: int = 8) -> List[Tuple[int, int]]:
    """Split [0, n) into `world` contiguous slices whose starts are multiples
    of `align` (the tcgen05 kernel needs 16-byte aligned row strides)."""
    if n < 1 or world < 1:
        raise ValueError("n and world must be >= 1")
    units = (n + align - 1) // align
    base, extra = divmod(units, world)
    bounds, start = [], 0
    for r in range(world):
        u = base + (1 if r < extra else 0)
        end = min(n, start + u * align)
        bounds.append((start, end))
        start = end
    return bounds


def globalize_location(loc_local: int, n0: int) -> int:
    """Slice-local located column -> global column (-1 stays -1)."""
    return -1 if loc_local < 0 else loc_local + n0


def shard_trials(trials: int, world: int, rank: int) -> range:
    """Contiguous, restartable trial range of one rank (seed-addressed)."""
    base, extra = divmod(trials, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def allreduce_counts(counts, group=None):
    """Sum the int64 counters {rows, detected, located, nan, ...} over ranks —
    the path's only collective (NCCL on GPU, gloo in the CPU tests)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def merge_counts(parts: Iterable[Sequence[int]]) -> List[int]:
    tot = None
    for p in parts:
        tot = list(p) if tot is None else [a + b for a, b in zip(tot, p)]
    return tot or []


# ------------------------------------------------------- device executors
class ShardedGemmBatch:
    """This rank's share of a batch of independent fused V-ABFT GEMMs.

    shapes: the whole batch [(m, k, n), ...] (e.g. 32 LLaMA-7B layers x 7
    GEMMs = 224); plan_gemm_batch assigns each GEMM to one rank, and this
    rank builds a FusedAbftGemm (per-weight B-side state) for each of its
    GEMMs only, from weight(i) -> K x N device tensor. A call runs every owned
    GEMM through the fused kernel on the current stream, accumulating the
    verdict counters; no operand crosses ranks. all_reduce() is the batch's
    only collective (proj/src/parallel.cpp:20-53 is the reference's
    trial-level equivalent)."""

    def __init__(self, shapes, weight, rank: int = 0, world: int = 1, **fused_kw):
        from .fused import FusedAbftGemm
        self.shapes = list(shapes)
        self.owned = plan_gemm_batch(self.shapes, world)[rank]
        self.gemms = {i: FusedAbftGemm(weight(i), **fused_kw) for i in self.owned}

    def flops(self) -> float:
        return float(sum(2 * self.shapes[i][0] * self.shapes[i][1] * self.shapes[i][2] for i in self.owned))

    def __call__(self, activation, out, counts) -> None:
        """activation(i) -> M x K input of GEMM i, out(i) -> M x N output."""
        for i in self.owned:
            self.gemms[i](activation(i), out=out(i), counts=counts)

    def close(self) -> None:
        for g in self.gemms.values():
            g.close()


class ColumnShardedGemm:
    """One GEMM split along N: this rank owns columns [n0, n1) of B and C and
    verifies them as an independent ABFT unit (thresholds with n = n1 - n0 from
    slice-local B statistics, checksum weights j + 1 over the slice), so its
    verdicts equal the reference's on (A, B[:, n0:n1]); located columns are
    shifted to global indices. A is replicated; nothing is exchanged but the
    counters."""

    def __init__(self, b_slice, n0: int, n_total: int, **fused_kw):
        from .fused import FusedAbftGemm
        self.n0, self.n_total = int(n0), int(n_total)
        self.g = FusedAbftGemm(b_slice, **fused_kw)

    @staticmethod
    def for_rank(B_full_slice_fn, n: int, rank: int, world: int, **fused_kw) -> "ColumnShardedGemm":
        n0, n1 = shard_columns(n, world)[rank]
        return ColumnShardedGemm(B_full_slice_fn(n0, n1), n0, n, **fused_kw)

    def __call__(self, A, out=None, counts=None, **kw):
        r = self.g(A, out=out, counts=counts, **kw)
        return r

    def global_location(self, r):
        """Slice-local located columns -> global columns (-1 stays -1)."""
        import torch
        return torch.where(r.location >= 0, r.location + self.n0, r.location)

    def close(self) -> None:
        self.g.close()
