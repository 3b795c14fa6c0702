"""Fault-injection campaigns on the GPU — injection_campaign
(proj/src/faults.cpp:170-216) re-designed for B200.

The reference runs one trial per (A, B) pair on the CPU: fresh operands,
encode, thresholds, one bit flip at a uniformly random eligible element of
C_accum (online) or C (offline), verify, tally the flipped row. Verification
is row-independent, so here EVERY ROW of one fused GEMM launch is an
independent trial: each row gets one planned fault (random column, fixed bit,
direction), injected inside the tcgen05 epilogue into the FP32 accumulator
(online) or the quantized output bits (offline) before the row sums, and
the fused verify tail produces the row's verdict. One launch = M trials.

Outcome counters follow CampaignOutcome (faults.hpp:68-85): applicable,
detected, located_correctly, nonfinite_after, with the same rates. For
multi-GPU campaigns each rank runs a seed-addressed trial range and the
counters are all-reduced (sharding.allreduce_counts).

Sampling note: the reference draws the position uniformly over the
eligible elements of one matrix; here the column is uniform per row and a
trial whose bit already holds the target value is not applicable. Given
the matrix, the conditional distribution over eligible positions is the
same uniform one, so detection/localization rates estimate the same
quantities.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import torch

from . import _capi
from .fused import FusedAbftGemm
from .sharding import allreduce_counts

_REC_BYTES = 24  # sizeof(vabft_fault_record)


def sample_matrix(shape, dist: str, gen: torch.Generator, device, dtype=torch.bfloat16) -> torch.Tensor:
    """Device sampler for the reference's distributions (distribution.cpp:44-52);
    values are quantized to the format by the final cast (RNE)."""
    name, _, rest = dist.partition(":")
    args = [float(t) for t in rest.split(",") if t] if rest else []
    wd = torch.float64 if dtype == torch.float64 else torch.float32  # draw in FP64 for FP64 operands
    arg = lambda i, d: args[i] if i < len(args) else d  # noqa: E731
    if name == "normal":
        x = torch.randn(shape, generator=gen, device=device, dtype=wd) * arg(1, 1.0) + arg(0, 0.0)
    elif name == "uniform":
        a, b = arg(0, -1.0), arg(1, 1.0)
        x = torch.rand(shape, generator=gen, device=device, dtype=wd) * (b - a) + a
    elif name == "truncnormal":
        mu, sd, lo, hi = arg(0, 0.0), arg(1, 1.0), arg(2, -1.0), arg(3, 1.0)
        x = torch.randn(shape, generator=gen, device=device, dtype=wd) * sd + mu
        bad = (x < lo) | (x > hi)
        while bool(bad.any()):
            x[bad] = torch.randn(int(bad.sum()), generator=gen, device=device, dtype=wd) * sd + mu
            bad = (x < lo) | (x > hi)
    elif name == "absnormal":
        x = (torch.randn(shape, generator=gen, device=device, dtype=wd) * arg(1, 1.0) + arg(0, 1.0)).abs()
    else:
        raise _capi.InvalidArgument(f"unknown distribution: {dist}")
    return x.to(dtype)


@dataclass
class CampaignOutcome:
    trials: int = 0
    applicable: int = 0
    detected: int = 0
    located_correctly: int = 0
    nonfinite_after: int = 0

    def detection_rate(self) -> float:
        return self.detected / self.applicable if self.applicable else 0.0

    def localization_accuracy(self) -> float:
        return self.located_correctly / self.detected if self.detected else 0.0

    def as_dict(self):
        return {"trials": self.trials, "applicable": self.applicable, "detected": self.detected,
                "located_correctly": self.located_correctly, "nonfinite_after": self.nonfinite_after,
                "detection_rate": self.detection_rate() if self.applicable else None,
                "localization_accuracy": self.localization_accuracy() if self.detected else None}


class DeviceCampaign:
    """M trials per fused launch; operands re-drawn every `refresh` launches."""

    def __init__(self, m: int, k: int, n: int, dist: str = "normal:1e-6,1", mode: str = "online",
                 threshold: str = "vabft", e_max: Optional[float] = None, direction: int = _capi.SET0TO1,
                 seed: int = 0, dtype=torch.bfloat16, device=None, refresh: int = 1):
        self.m, self.k, self.n = m, k, n
        self.dist, self.mode, self.direction = dist, mode, direction
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.gen = torch.Generator(device=self.device)
        self.gen.manual_seed(seed)
        self.dtype = dtype
        self.refresh = max(1, refresh)
        self.B = sample_matrix((k, n), dist, self.gen, self.device, dtype)
        self.A = sample_matrix((m, k), dist, self.gen, self.device, dtype)
        self.g = FusedAbftGemm(self.B, mode=mode, threshold=threshold, e_max=e_max)
        self.rec = torch.empty(m * _REC_BYTES, dtype=torch.uint8, device=self.device)
        self.launches = 0

    def _redraw(self):
        self.B = sample_matrix((self.k, self.n), self.dist, self.gen, self.device, self.dtype)
        self.A = sample_matrix((self.m, self.k), self.dist, self.gen, self.device, self.dtype)
        self.g.update_weight(self.B)

    def launch(self, bit: int, totals: torch.Tensor) -> None:
        """One fused launch = M trials; adds [trials, applicable, detected,
        located, nonfinite] into the device tensor `totals` (no host sync)."""
        if self.launches and self.launches % self.refresh == 0:
            self._redraw()
        self.launches += 1
        m, dev = self.m, self.device
        col = torch.randint(0, self.n, (m,), generator=self.gen, device=dev, dtype=torch.int32)
        bits = torch.full((m,), bit, dtype=torch.int32, device=dev)
        dirs = torch.full((m,), self.direction, dtype=torch.int32, device=dev)
        r = self.g(self.A, faults={"col": col, "bit": bits, "dir": dirs, "records": self.rec})
        recs = self.rec.view(m, _REC_BYTES)
        after = recs[:, 8:16].contiguous().view(torch.float64).view(m)
        applied = recs[:, 16:20].contiguous().view(torch.int32).view(m) != 0
        det = (r.detected != 0) & applied
        located = det & (r.location == col.to(torch.int64))
        nonfinite = applied & ~torch.isfinite(after)
        totals += torch.stack([torch.tensor(m, device=dev, dtype=torch.int64), applied.sum(), det.sum(),
                               located.sum(), nonfinite.sum()]).to(torch.int64)

    def launch_operand_a(self, bit: int, totals: torch.Tensor) -> None:
        """M trials: one fault per row i in A[i][k_i] (bits of the BF16/FP16
        operand) as the tensor cores read it; checksums from the clean A.
        The error spreads over row i, so only detection is tallied (located
        stays 0)."""
        if self.launches and self.launches % self.refresh == 0:
            self._redraw()
        self.launches += 1
        m, dev = self.m, self.device
        k_idx = torch.randint(0, self.k, (m,), generator=self.gen, device=dev, dtype=torch.int32)
        bits = torch.full((m,), bit, dtype=torch.int32, device=dev)
        dirs = torch.full((m,), self.direction, dtype=torch.int32, device=dev)
        r = self.g(self.A, faults={"target": "A", "col": k_idx, "bit": bits, "dir": dirs, "records": self.rec})
        recs = self.rec.view(m, _REC_BYTES)
        after = recs[:, 8:16].contiguous().view(torch.float64).view(m)
        applied = recs[:, 16:20].contiguous().view(torch.int32).view(m) != 0
        det = (r.detected != 0) & applied
        nonfinite = applied & ~torch.isfinite(after)
        z = torch.zeros((), dtype=torch.int64, device=dev)
        totals += torch.stack([torch.tensor(m, device=dev, dtype=torch.int64), applied.sum(), det.sum(), z,
                               nonfinite.sum()]).to(torch.int64)

    def launch_operand_b(self, bit: int, totals: torch.Tensor) -> None:
        """One trial: one fault in B[k][j] (every row's column j is hit).
        Detected = some row flags it; located = every flagging row points at
        column j."""
        from .fused import operand_faults
        if self.launches and self.launches % self.refresh == 0:
            self._redraw()
        self.launches += 1
        dev = self.device
        k = int(torch.randint(0, self.k, (1,), generator=self.gen, device=dev).item())
        j = int(torch.randint(0, self.n, (1,), generator=self.gen, device=dev).item())
        rec = self.rec[:_REC_BYTES]
        r = self.g(self.A, faults={"target": "B", "operand": operand_faults([(k, j, bit, self.direction)], dev),
                                   "records": rec})
        after = rec[8:16].view(torch.float64)
        applied = rec[16:20].view(torch.int32)[0] != 0
        det_rows = r.detected != 0
        det = applied & det_rows.any()
        located = det & (r.location[det_rows] == j).all()
        nonfinite = applied & ~torch.isfinite(after[0])
        totals += torch.stack([torch.ones((), dtype=torch.int64, device=dev), applied.long(), det.long(),
                               located.long(), nonfinite.long()])

    def run(self, bit: int, trials: int, reduce: bool = True, target: str = "output") -> CampaignOutcome:
        """target: "output" (accumulator online / output offline, M trials per
        launch), "A" (operand A, M trials per launch), "B" (operand B, one
        trial per launch)."""
        totals = torch.zeros(5, dtype=torch.int64, device=self.device)
        if target == "B":
            for _ in range(trials):
                self.launch_operand_b(bit, totals)
        else:
            step = self.launch if target == "output" else self.launch_operand_a
            for _ in range(math.ceil(trials / self.m)):
                step(bit, totals)
        if reduce:
            allreduce_counts(totals)
        t = totals.tolist()
        return CampaignOutcome(*t)

    def close(self):
        self.g.close()
