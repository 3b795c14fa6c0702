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

from typing import Sequence

import torch

from .campaign import sample_matrix
from .emax import CalibrationModel, CalibrationResult, fit_model  # noqa: F401 (re-exported)
from .fused import FusedAbftGemm


def calibrate(fmt: str = "bf16", sizes: Sequence[int] = (128, 256, 512, 1024, 2048, 4096), trials: int = 20,
              mode: str = "online", seed: int = 0, dist: str = "absnormal:1,1") -> CalibrationResult:
    """calibrate (calibration.cpp:88-150) on the fused device path. fmt
    "tf32" calibrates FP32 operands on the single-pass TF32 kernel."""
    passes = 1 if fmt == "tf32" else 3
    dtype = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32, "tf32": torch.float32,
             "fp64": torch.float64}[fmt]
    dev = torch.device("cuda", torch.cuda.current_device())
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    maxima, aborted = [], 0
    for s in sizes:
        mx = 0.0
        for _ in range(trials):
            A = sample_matrix((s, s), dist, gen, dev, dtype)
            B = sample_matrix((s, s), dist, gen, dev, dtype)
            g = FusedAbftGemm(B, mode=mode, e_max=1.0, tf32_passes=passes)
            r = g(A, checksums=True)
            rel = (r.diff1.abs() / r.row_check1.abs())
            if not bool(torch.isfinite(rel).all()):
                aborted += 1
            else:
                mx = max(mx, float(rel.max().item()))
            g.close()
        maxima.append(mx)
    return CalibrationResult.from_maxima(fmt, mode, sizes, maxima, trials, aborted)
