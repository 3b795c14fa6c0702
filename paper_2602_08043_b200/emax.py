"""e_max models: the reference's calibration result type (fit_model /
CalibrationResult::e_max_for, proj/src/calibration.cpp:15-74) and the
device-calibrated defaults the fused tcgen05 path uses.

The reference resolves e_max per run by calibrating (harness.cpp
resolve_run_e_max: calibrate(precision, mode, {128, 256, 512, K}) then
e_max_for(K)). Online verification compares the FP32 accumulator of the
tensor core, whose rounding the CPU emulator does not reproduce, so the
online defaults here come from the same protocol run on the B200 fused path
(calibration.calibrate; raw data in profiles/r02_calibration_device_100trials.jsonl):
|N(1,1)| square operands, per size the max over trials and rows of
|D1| / |row_check1|. Offline defaults are the reference's format constants
(precision.cpp:44-62), which its own calibration reproduces (the 2u floor).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple


@dataclass
class CalibrationModel:
    kind: str = "constant"  # "constant" | "sqrt_scaled" (EmaxModel::Kind)
    value: float = 0.0
    scale: float = 0.0
    offset: float = 0.0
    cv: float = 0.0
    r2: float = 0.0


def _seq_sum(xs) -> float:
    """Left-to-right FP64 sum (the reference's loops). Python 3.12's built-in
    sum() of floats is compensated (Neumaier), which rounds differently."""
    t = 0.0
    for x in xs:
        t += x
    return t


def fit_model(sizes: Sequence[int], maxima: Sequence[float]) -> CalibrationModel:
    """fit_model (calibration.cpp:15-59): Constant if the maxima vary little
    (CV < 15%), else least squares of max against sqrt(size). Same
    operations in the same order as the reference (bit-identical results)."""
    if len(sizes) != len(maxima) or not sizes:
        raise ValueError("fit_model: sizes and maxima must match and be nonempty")
    n = len(maxima)
    m = CalibrationModel()
    mean = _seq_sum(maxima) / n
    m.value = mean
    if n >= 2 and mean > 0.0:
        ss = _seq_sum((v - mean) * (v - mean) for v in maxima)
        m.cv = math.sqrt(ss / (n - 1)) / mean
    if n >= 2:
        sx = sy = sxx = sxy = 0.0
        for s_, y in zip(sizes, maxima):
            x = math.sqrt(float(s_))
            sx += x
            sy += y
            sxx += x * x
            sxy += x * y
        denom = n * sxx - sx * sx
        if denom != 0.0:
            m.scale = (n * sxy - sx * sy) / denom
            m.offset = (sy - m.scale * sx) / n
            ss_res = ss_tot = 0.0
            for s_, y in zip(sizes, maxima):
                fit = m.scale * math.sqrt(float(s_)) + m.offset
                ss_res += (y - fit) * (y - fit)
                ss_tot += (y - mean) * (y - mean)
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

    @classmethod
    def from_maxima(cls, precision: str, mode: str, sizes: Sequence[int], maxima: Sequence[float],
                    trials: int, aborted: int = 0) -> "CalibrationResult":
        """calibrate()'s result assembly (calibration.cpp:135-150)."""
        u = unit_roundoff_for(precision, mode)
        overall = max(maxima) if maxima else 0.0
        return cls(precision, mode, list(sizes), list(maxima), fit_model(list(sizes), list(maxima)),
                   max(1.2 * overall, 2.0 * u), u, trials, aborted)

    def e_max_for(self, dim: int) -> float:
        """e_max_for (calibration.cpp:61-74): margin 1.2, floor 2u; a
        SqrtScaled model is inflated so every calibrated size stays covered."""
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


def unit_roundoff_for(precision: str, mode: str) -> float:
    """u of the verification precision: the FP32 accumulator online, the
    format itself offline (checksum_precision_for, checksum.cpp:18-24)."""
    if precision == "tf32":  # FP32 operands on one TF32 pass: the products carry TF32 rounding
        return 2.0 ** -11
    if mode == "online":
        return 2.0 ** -53 if precision == "fp64" else 2.0 ** -24
    return {"bf16": 2.0 ** -8, "fp16": 2.0 ** -11, "fp32": 2.0 ** -24, "fp64": 2.0 ** -53}[precision]


# Device calibration of the fused paths (B200, calibration.calibrate: the
# reference protocol of calibration.cpp:88-150; tools/calib_run.py): per
# square size the maximum of |D1| / |row_check1| over two campaigns, 100 and
# 1000 trials per size (profiles/r02_calibration_device_100trials.jsonl,
# profiles/r02_calibration_device_1000trials.jsonl) — 1100 trials per size,
# ~3.7x the reference's default of 300 (harness.hpp:37).
DEVICE_CALIBRATION: Dict[Tuple[str, str], Tuple[List[int], List[float]]] = {
    # the tcgen05 FP32 accumulator, BF16 operands
    ("bf16", "online"): ([128, 256, 512, 1024, 2048, 4096, 8192, 16384],
                         [1.179e-06, 1.166e-06, 1.564e-06, 2.728e-06, 6.234e-06, 1.520e-05, 3.663e-05, 8.456e-05]),
    # FP16 operands on the same accumulator. (FP16 OFFLINE is not tabled: with
    # |N(1,1)| operands the FP16-quantized checksums saturate at 65504 from
    # size 256 on, so the protocol measures overflow, not rounding; the format
    # constant stays. BF16 offline maxima, 3.0e-3 .. 4.0e-3, sit below the 2u
    # floor 7.8e-3, which the format constant 8e-3 covers.)
    ("fp16", "online"): ([128, 256, 512, 1024, 2048, 4096, 8192, 16384],
                         [1.601e-06, 2.175e-06, 3.641e-06, 6.823e-06, 1.359e-05, 2.733e-05, 5.487e-05, 1.097e-04]),
    # FP64 SIMT DFMA path (sequential FMA accumulation, FP64 blocked:128
    # checksums; online == offline)
    ("fp64", "online"): ([128, 256, 512, 1024, 2048, 4096, 8192, 16384],
                         [2.174e-15, 1.532e-15, 1.196e-15, 9.962e-16, 9.945e-16, 1.454e-15, 1.650e-15, 2.616e-15]),
    # FP32 on tcgen05 with 3xTF32: the products are FP32-accurate but the
    # tensor core's FP32 accumulation truncates, so |D1|/|r| grows linearly in
    # n (as for BF16 online)
    ("fp32", "online"): ([128, 256, 512, 1024, 2048, 4096, 8192, 16384],
                         [2.335e-06, 3.537e-06, 6.741e-06, 1.287e-05, 2.541e-05, 5.055e-05, 9.943e-05, 1.902e-04]),
    # one TF32 pass: TF32 operand rounding dominates, flat in n; the 2u floor
    # (u = 2^-11) applies
    ("tf32", "online"): ([128, 256, 512, 1024, 2048, 4096, 8192, 16384],
                         [4.617e-04, 4.300e-04, 4.103e-04, 4.004e-04, 3.973e-04, 4.045e-04, 4.299e-04, 4.893e-04]),
}

# reference format defaults (PrecisionSpec::bf16/fp16, precision.cpp:44-62)
FORMAT_DEFAULT = {"bf16": 8e-3, "fp16": 1e-3}
# sqrt-scaled format models a*sqrt(dim) + b (PrecisionSpec::fp32/fp64, precision.cpp:64-82)
FORMAT_MODEL = {"fp32": (5e-9, 1.2e-7), "fp64": (1e-17, 2.5e-16),
                # single-pass TF32 (no reference format): 4 u of TF32 until calibrated
                "tf32": (0.0, 4 * 2.0 ** -11)}


def device_calibration(precision: str, mode: str) -> CalibrationResult:
    key = (precision, mode)
    if key not in DEVICE_CALIBRATION:
        raise KeyError(f"no device calibration for {precision}/{mode}")
    sizes, maxima = DEVICE_CALIBRATION[key]
    return CalibrationResult.from_maxima(precision, mode, sizes, maxima, trials=1100)


def measured_max(precision: str, mode: str, size: int) -> float:
    """The calibration maximum at `size`: the device table, log-log
    interpolated between calibrated sizes (extrapolated along the end
    segments outside them)."""
    sizes, maxima = DEVICE_CALIBRATION[(precision, mode)]
    if size in sizes:
        return maxima[sizes.index(size)]
    i = 1
    while i < len(sizes) - 1 and sizes[i] < size:
        i += 1
    x0, x1 = math.log(sizes[i - 1]), math.log(sizes[i])
    y0, y1 = math.log(maxima[i - 1]), math.log(maxima[i])
    return math.exp(y0 + (y1 - y0) * (math.log(size) - x0) / (x1 - x0))


def resolve_run_e_max(precision: str, mode: str, k: int) -> float:
    """resolve_run_e_max (harness.cpp, with auto_calib_sizes): calibration
    sizes {128, 256, 512} plus K (K > 512) or with K prepended (K < 128),
    model fitted on those, e_max_for(K) — with the device calibration's
    maxima standing in for per-run trials."""
    sizes = [128, 256, 512]
    if k > 512:
        sizes.append(k)
    if k < 128:
        sizes.insert(0, k)
    maxima = [measured_max(precision, mode, s) for s in sizes]
    return CalibrationResult.from_maxima(precision, mode, sizes, maxima, trials=1100).e_max_for(k)


def default_e_max(precision: str, mode: str, k: int) -> float:
    """e_max the fused path uses when the caller gives none: calibrate()'s
    `recommended` rule applied at the accumulation length itself,
    max(1.2 x max(K), 2u), with max(K) from the device calibration.
    (resolve_run_e_max above is the reference's per-run rule; its lambda
    inflation turns erratic when the sqrt fit nearly vanishes at a small
    calibration size, e.g. 1.6e-3 at K = 3072 against 1.8e-5 at K = 4096.)
    The FP16 online path shares the BF16 path's FP32 accumulator and uses
    its table when it has none of its own; offline without a table, the
    format constant."""
    key = (precision, mode) if (precision, mode) in DEVICE_CALIBRATION else None
    if key is None and mode == "online" and precision == "fp16":
        key = ("bf16", "online")
    if key is None and precision in ("fp32", "tf32", "fp64"):
        # the wide formats verify in their own precision: online == offline
        other = (precision, "offline" if mode == "online" else "online")
        key = other if other in DEVICE_CALIBRATION else None
    if key is None:
        if precision in FORMAT_MODEL:
            a, b = FORMAT_MODEL[precision]
            return a * math.sqrt(k) + b
        return FORMAT_DEFAULT[precision]
    return max(1.2 * measured_max(key[0], key[1], k), 2.0 * unit_roundoff_for(precision, mode))
