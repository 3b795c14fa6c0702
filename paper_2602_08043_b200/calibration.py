"""e_max calibration on the B200 — calibrate / fit_model / e_max_for
(proj/src/calibration.cpp:15-150), run on the device path
whose rounding the thresholds must cover.

Protocol (the reference's): square |N(1,1)| matrices of each size, per trial
the max over rows of |D1| / |row_check1|; per size the max over trials;
model = Constant if the maxima vary little (CV < 15%) else a least-squares
fit of max against sqrt(size); recommended = max(1.2 x overall max, 2u) with
u the unit roundoff of the verification precision (FP32 for online mode).

For the TENSOR engine the measured quantity is exactly what the fused kernel
compares against T: the FP32 (tcgen05) accumulator's blocked:128 row sums
versus the FP32 blocked:128 checksums, so online e_max reflects the tensor
core's accumulation, not the CPU emulator's.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Sequence

import torch

from .campaign import sample_matrix
from .fused import FusedAbftGemm


@dataclass
class CalibrationModel:
    kind: str = "constant"  # "constant" | "sqrt_scaled"
    value: float = 0.0
    scale: float = 0.0
    offset: float = 0.0
    cv: float = 0.0
    r2: float = 0.0


def fit_model(sizes: Sequence[int], maxima: Sequence[float]) -> CalibrationModel:
    """fit_model (calibration.cpp:15-59)."""
    if len(sizes) != len(maxima) or not sizes:
        raise ValueError("fit_model: sizes and maxima must match and be nonempty")
    n = len(maxima)
    m = CalibrationModel()
    mean = sum(maxima) / n
    m.value = mean
    if n >= 2 and mean > 0.0:
        ss = sum((v - mean) ** 2 for v in maxima)
        m.cv = math.sqrt(ss / (n - 1)) / mean
    if n >= 2:
        xs = [math.sqrt(float(s)) for s in sizes]
        sx, sy = sum(xs), sum(maxima)
        sxx = sum(x * x for x in xs)
        sxy = sum(x * y for x, y in zip(xs, maxima))
        denom = n * sxx - sx * sx
        if denom != 0.0:
            m.scale = (n * sxy - sx * sy) / denom
            m.offset = (sy - m.scale * sx) / n
            ss_res = sum((y - (m.scale * x + m.offset)) ** 2 for x, y in zip(xs, maxima))
            ss_tot = sum((y - mean) ** 2 for y in maxima)
            m.r2 = 1.0 - ss_res / ss_tot if ss_tot > 0.0 else 1.0
    m.kind = "constant" if (n < 2 or m.cv < 0.15 or m.scale <= 0.0) else "sqrt_scaled"
    return m


@dataclass
class CalibrationResult:
    precision: str
    mode: str
    sizes: List[int]
    maxima: List[float]
    model: CalibrationModel
    recommended: float
    unit_roundoff: float
    trials_per_size: int
    aborted_trials: int = 0
    engine: str = "tensor"

    def e_max_for(self, dim: int) -> float:
        """e_max_for (calibration.cpp:61-74)."""
        floor = 2.0 * self.unit_roundoff
        if self.model.kind == "constant":
            return max(self.recommended, floor)
        lam = 1.0
        for s, mx in zip(self.sizes, self.maxima):
            fit = self.model.scale * math.sqrt(float(s)) + self.model.offset
            if fit > 0.0:
                lam = max(lam, mx / fit)
        return max(1.2 * lam * (self.model.scale * math.sqrt(float(dim)) + self.model.offset), floor)

    def as_dict(self):
        return {"precision": self.precision, "mode": self.mode, "engine": self.engine, "sizes": self.sizes,
                "maxima": self.maxima, "model": self.model.__dict__, "recommended": self.recommended,
                "trials": self.trials_per_size, "aborted_trials": self.aborted_trials}


def calibrate(fmt: str = "bf16", sizes: Sequence[int] = (128, 256, 512, 1024, 2048, 4096), trials: int = 20,
              mode: str = "online", seed: int = 0, dist: str = "absnormal:1,1") -> CalibrationResult:
    """calibrate (calibration.cpp:88-150) on the fused tcgen05 path."""
    dtype = torch.bfloat16 if fmt == "bf16" else torch.float16
    dev = torch.device("cuda", torch.cuda.current_device())
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    maxima, aborted = [], 0
    for s in sizes:
        mx = 0.0
        for _ in range(trials):
            A = sample_matrix((s, s), dist, gen, dev, dtype)
            B = sample_matrix((s, s), dist, gen, dev, dtype)
            g = FusedAbftGemm(B, mode=mode, e_max=1.0)
            r = g(A, checksums=True)
            rel = (r.diff1.abs() / r.row_check1.abs())
            if not bool(torch.isfinite(rel).all()):
                aborted += 1
            else:
                mx = max(mx, float(rel.max().item()))
            g.close()
        maxima.append(mx)
    u = 2.0 ** -24 if mode == "online" else (2.0 ** -8 if fmt == "bf16" else 2.0 ** -11)
    model = fit_model(list(sizes), maxima)
    overall = max(maxima) if maxima else 0.0
    return CalibrationResult(fmt, mode, list(sizes), maxima, model, max(1.2 * overall, 2.0 * u), u, trials, aborted)
