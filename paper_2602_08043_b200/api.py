"""Python mirror of the reference's C++ API (namespace vabft,
proj/include/vabft/*.hpp) on top of the C-ABI.

Same names, argument meaning and error behaviour as the reference; host
matrices are numpy FP64 arrays holding values on the format grid (the
reference's vabft::Matrix storage) and results come back by value. Every
numerical step runs on the GPU through libvabft_b200.so; the scalar helpers
(quantize, threshold_row, localize, encode/decode_bits, aabft_sigma,
resolve_e_max) call the library's host implementations.

Errors map to the reference's exception classes:
  std::invalid_argument -> _capi.InvalidArgument (a ValueError)
  std::domain_error     -> _capi.DomainError     (a ValueError)
  std::range_error      -> _capi.RangeError
  std::out_of_range     -> _capi.OutOfRange      (an IndexError)
  std::logic_error      -> _capi.LogicError
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace
from typing import Optional, Sequence

import numpy as np
import torch

from . import _capi
from ._capi import check, lib
from .device import fmt_name, ptr, stream_ptr, to_device, to_host

Format = _capi.FORMAT_CODES


class AccumKind:
    FP32_ACCUM_ROUND_OUTPUT = _capi.ACCUM_FP32_ROUND_OUTPUT
    NATIVE_SEQUENTIAL = _capi.ACCUM_SEQUENTIAL
    NATIVE_BLOCKED = _capi.ACCUM_BLOCKED
    NATIVE_PAIRWISE = _capi.ACCUM_PAIRWISE


class VerifyMode:
    OFFLINE = "offline"
    ONLINE = "online"


class FlipDirection:
    FLIP = _capi.FLIP
    SET0TO1 = _capi.SET0TO1
    SET1TO0 = _capi.SET1TO0
    ANY = _capi.ANY


def _mode_code(mode) -> int:
    if mode in ("offline", _capi.OFFLINE):
        return _capi.OFFLINE
    if mode in ("online", _capi.ONLINE):
        return _capi.ONLINE
    raise _capi.InvalidArgument(f"unknown mode: {mode}")


# ------------------------------------------------------------- precision
@dataclass(frozen=True)
class AccumStrategy:
    """vabft::AccumStrategy (precision.hpp:28-33)."""
    kind: int = AccumKind.NATIVE_SEQUENTIAL
    block_len: int = 128

    def describe(self) -> str:
        return {0: "fp32-accum", 1: "sequential", 2: f"blocked:{self.block_len}", 3: "pairwise"}[self.kind]


@dataclass(frozen=True)
class EmaxModel:
    """vabft::EmaxModel (precision.hpp:36-47)."""
    kind: int = 0  # 0 Constant, 1 SqrtScaled
    scale: float = 0.0
    offset: float = 0.0

    @staticmethod
    def constant(v: float) -> "EmaxModel":
        return EmaxModel(0, 0.0, v)

    @staticmethod
    def sqrt_scaled(scale: float, offset: float) -> "EmaxModel":
        return EmaxModel(1, scale, offset)

    def resolve(self, dim: int) -> float:
        return self.offset if self.kind == 0 else self.scale * math.sqrt(float(dim)) + self.offset


@dataclass(frozen=True)
class PrecisionSpec:
    """vabft::PrecisionSpec (precision.hpp:54-85)."""
    format: str
    mantissa_bits: int
    unit_roundoff: float
    accumulation: AccumStrategy
    e_max_model: EmaxModel
    overflow_error: bool = False

    @staticmethod
    def of(fmt) -> "PrecisionSpec":
        p = _capi.precision(fmt_name(fmt))
        return PrecisionSpec(fmt_name(fmt), p.mantissa_bits, p.unit_roundoff,
                             AccumStrategy(p.accumulation.kind, p.accumulation.block_len),
                             EmaxModel(p.emax_kind, p.emax_scale, p.emax_offset), bool(p.overflow))

    @staticmethod
    def bf16():
        return PrecisionSpec.of("bf16")

    @staticmethod
    def fp16():
        return PrecisionSpec.of("fp16")

    @staticmethod
    def fp32():
        return PrecisionSpec.of("fp32")

    @staticmethod
    def fp64():
        return PrecisionSpec.of("fp64")

    def with_accumulation(self, s: AccumStrategy) -> "PrecisionSpec":
        return replace(self, accumulation=s)

    def with_e_max(self, m: EmaxModel) -> "PrecisionSpec":
        return replace(self, e_max_model=m)

    @property
    def code(self) -> int:
        return _capi.FORMAT_CODES[self.format]

    def bit_width(self) -> int:
        return {"bf16": 16, "fp16": 16, "fp32": 32, "fp64": 64}[self.format]

    def name(self) -> str:
        return self.format

    def to_c(self) -> _capi.Precision:
        p = _capi.Precision()
        p.format = self.code
        p.mantissa_bits = self.mantissa_bits
        p.unit_roundoff = self.unit_roundoff
        p.accumulation.kind = self.accumulation.kind
        p.accumulation.block_len = self.accumulation.block_len
        p.emax_kind = self.e_max_model.kind
        p.emax_scale = self.e_max_model.scale
        p.emax_offset = self.e_max_model.offset
        p.overflow = int(self.overflow_error)
        return p


def _spec(spec) -> PrecisionSpec:
    return spec if isinstance(spec, PrecisionSpec) else PrecisionSpec.of(spec)


def quantize(x: float, spec) -> float:
    """quantize (precision.cpp:129-159)."""
    out = C.c_double()
    check(lib.vabft_quantize(float(x), C.byref(_spec(spec).to_c()), C.byref(out)))
    return out.value


def accumulates_in_float(spec) -> bool:
    """accumulates_in_float (precision.cpp:203-206)."""
    s = _spec(spec)
    return s.accumulation.kind == AccumKind.FP32_ACCUM_ROUND_OUTPUT or s.format == "fp32"


# -------------------------------------------------------------- checksum
def checksum_precision_for(spec, mode) -> PrecisionSpec:
    """checksum_precision_for (checksum.cpp:18-24)."""
    s = _spec(spec)
    if _mode_code(mode) == _capi.OFFLINE:
        return s
    base = PrecisionSpec.fp64() if s.format == "fp64" else PrecisionSpec.fp32()
    return base.with_accumulation(s.accumulation)


@dataclass
class EncodedProduct:
    """vabft::EncodedProduct (checksum.hpp:35-48)."""
    c: np.ndarray
    row_check1: np.ndarray
    row_check2: np.ndarray
    col_check1: np.ndarray
    col_check2: np.ndarray
    checksum_precision: PrecisionSpec
    mode: str
    c_accum: np.ndarray
    format: str = "fp64"
    engine: str = "exact"

    def verification_source(self) -> np.ndarray:
        return self.c_accum if self.mode == "online" else self.c

    def verification_format(self) -> str:
        if self.mode == "online":
            return "fp64" if self.format == "fp64" else "fp32"
        return self.format


_ENGINES = {"exact": _capi.ENGINE_EXACT, "tensor": _capi.ENGINE_TENSOR}


def encode_and_multiply(a: np.ndarray, b: np.ndarray, mode="offline", spec="fp64",
                        engine: str = "exact") -> EncodedProduct:
    """encode_and_multiply (checksum.cpp:150-158) on the GPU.

    engine="exact": order-exact kernels, bit-identical to the reference.
    engine="tensor": tcgen05 GEMM (BF16/FP16) or the SIMT DFMA GEMM (FP64),
    checksums in blocked:128 order.
    """
    s = _spec(spec)
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise _capi.InvalidArgument("gemm_emulated: inner dimensions disagree")
    m, k = a.shape
    n = b.shape[1]
    mc = _mode_code(mode)
    dA, dB = to_device(a, s.format), to_device(b, s.format)
    dC = torch.empty((m, n), dtype=dA.dtype, device="cuda")
    acc_dtype = torch.float64 if (s.format == "fp64" and not accumulates_in_float(s)) else torch.float32
    dCa = torch.empty((m, n), dtype=acc_dtype, device="cuda")
    r1, r2 = (torch.empty(m, dtype=torch.float64, device="cuda") for _ in range(2))
    c1, c2 = (torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2))
    check(lib.vabft_encode_and_multiply(C.byref(s.to_c()), mc, _ENGINES[engine], m, n, k, ptr(dA), ptr(dB),
                                        ptr(dC), ptr(dCa), ptr(r1), ptr(r2), ptr(c1), ptr(c2), None, 0,
                                        stream_ptr()))
    torch.cuda.synchronize()
    cs = checksum_precision_for(s, mode)
    if engine == "tensor":
        # FP32 arithmetic (FP64 for FP64), blocked:128 order, in both modes
        base = PrecisionSpec.fp64() if s.format == "fp64" else PrecisionSpec.fp32()
        cs = base.with_accumulation(AccumStrategy(AccumKind.NATIVE_BLOCKED, 128))
    out = EncodedProduct(to_host(dC), to_host(r1), to_host(r2), to_host(c1), to_host(c2), cs,
                         "online" if mc else "offline", to_host(dCa), s.format, engine)
    if mc == _capi.OFFLINE:
        for v in (out.row_check1, out.row_check2, out.col_check1, out.col_check2):
            if not np.all(np.isfinite(v)):
                raise _capi.DomainError("quantize: non-finite input")
    return out


def row_sums(c: np.ndarray, sum_precision, src_format: Optional[str] = None):
    """row_sums (checksum.cpp:160-187); `c` holds values of `src_format`
    (default: the sum precision's format)."""
    sp = _spec(sum_precision)
    c = np.asarray(c, dtype=np.float64)
    m, n = c.shape
    sf = src_format or sp.format
    dC = to_device(c, sf)
    r1, r2 = (torch.empty(m, dtype=torch.float64, device="cuda") for _ in range(2))
    check(lib.vabft_row_sums(C.byref(sp.to_c()), _capi.FORMAT_CODES[sf], m, n, ptr(dC), ptr(r1), ptr(r2),
                             stream_ptr()))
    torch.cuda.synchronize()
    return to_host(r1), to_host(r2)


# ----------------------------------------------------------------- stats
@dataclass
class RowStats:
    """vabft::RowStats (stats.hpp:11-17)."""
    mean: float = 0.0
    max: float = 0.0
    min: float = 0.0
    var_bound: float = 0.0
    n: int = 0


def _row_stats_matrix(x: np.ndarray, fmt="fp64"):
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[None, :]
    rows, cols = x.shape
    if cols < 1:
        raise _capi.InvalidArgument("row_stats: empty row")
    d = to_device(x, fmt)
    outs = [torch.empty(rows, dtype=torch.float64, device="cuda") for _ in range(4)]
    check(lib.vabft_row_stats(_capi.FORMAT_CODES[fmt], rows, cols, ptr(d), *[ptr(o) for o in outs], stream_ptr()))
    return [to_host(o) for o in outs]


def row_stats(values: Sequence[float]) -> RowStats:
    """row_stats (stats.cpp:9-32) on the GPU."""
    v = np.asarray(values, dtype=np.float64)
    if v.size == 0:
        raise _capi.InvalidArgument("row_stats: empty row")
    mean, mx, mn, vb = _row_stats_matrix(v[None, :])
    return RowStats(float(mean[0]), float(mx[0]), float(mn[0]), float(vb[0]), int(v.size))


def precompute_b_stats(b: np.ndarray, fmt="fp64") -> list:
    """precompute_b_stats (threshold_vabft.cpp:8-13)."""
    b = np.asarray(b, dtype=np.float64)
    mean, mx, mn, vb = _row_stats_matrix(b, fmt)
    return [RowStats(float(mean[i]), float(mx[i]), float(mn[i]), float(vb[i]), b.shape[1]) for i in range(b.shape[0])]


@dataclass
class BStatsSummary:
    """vabft::BStatsSummary (threshold_vabft.hpp:28-34); sums in k order."""
    sum_abs_mean: float = 0.0
    sum_mean_sq: float = 0.0
    sum_var: float = 0.0
    k_len: int = 0

    @staticmethod
    def from_stats(stats: Sequence[RowStats]) -> "BStatsSummary":
        if len(stats) == 0:
            raise _capi.InvalidArgument("BStatsSummary: empty stats")
        s = BStatsSummary(k_len=len(stats))
        for r in stats:
            if r.var_bound < 0.0:
                raise _capi.LogicError("BStatsSummary: negative variance bound")
            s.sum_abs_mean += abs(r.mean)
            s.sum_mean_sq += r.mean * r.mean
            s.sum_var += r.var_bound
        return s


@dataclass
class VabftParams:
    """vabft::VabftParams (threshold_vabft.hpp:10-13)."""
    e_max: float = 0.0
    c_sigma: float = 2.5


@dataclass
class ThresholdBreakdown:
    det: float = 0.0
    var23: float = 0.0
    var4: float = 0.0
    total: float = 0.0


def threshold_row(a_stats: RowStats, b, n: int, params: VabftParams) -> ThresholdBreakdown:
    """threshold_row (threshold_vabft.cpp:28-47); `b` is a BStatsSummary or a list of RowStats."""
    if not isinstance(b, BStatsSummary):
        b = BStatsSummary.from_stats(b)
    a4 = (C.c_double * 4)(a_stats.mean, a_stats.max, a_stats.min, a_stats.var_bound)
    b3 = (C.c_double * 3)(b.sum_abs_mean, b.sum_mean_sq, b.sum_var)
    out = (C.c_double * 4)()
    check(lib.vabft_threshold_row(a4, b3, int(n), params.e_max, params.c_sigma, out))
    return ThresholdBreakdown(*out)


def resolve_e_max(spec, dim: int) -> float:
    """resolve_e_max (threshold_vabft.cpp:49-52)."""
    out = C.c_double()
    check(lib.vabft_resolve_e_max(C.byref(_spec(spec).to_c()), int(dim), C.byref(out)))
    return out.value


def vabft_thresholds(a: np.ndarray, b: np.ndarray, params: VabftParams, spec="fp64",
                     return_summary: bool = False):
    """vabft_thresholds (threshold_vabft.cpp:54-61) on the GPU."""
    s = _spec(spec)
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m, k = a.shape
    if b.shape[0] != k:
        raise _capi.InvalidArgument("vabft_thresholds: inner dimensions disagree")
    n = b.shape[1]
    dA, dB = to_device(a, s.format), to_device(b, s.format)
    T = torch.empty(m, dtype=torch.float64, device="cuda")
    summ = torch.empty(3, dtype=torch.float64, device="cuda")
    check(lib.vabft_vabft_thresholds(s.code, m, n, k, ptr(dA), ptr(dB), params.e_max, params.c_sigma, ptr(T),
                                     ptr(summ), stream_ptr()))
    out = to_host(T)
    return (out, to_host(summ)) if return_summary else out


# ---------------------------------------------------------------- A-ABFT
@dataclass
class AabftParams:
    """vabft::AabftParams (threshold_aabft.hpp:14-22)."""
    mantissa_bits: int = 53
    fixed_y: Optional[float] = 21.0
    confidence_multiplier: float = 3.0

    @staticmethod
    def for_format(fmt) -> "AabftParams":
        f = fmt_name(fmt) if not isinstance(fmt, PrecisionSpec) else fmt.format
        if f == "fp64":
            return AabftParams(53, 21.0)
        if f == "fp32":
            return AabftParams(23, 21.0)
        if f == "bf16":
            return AabftParams(8, None)
        return AabftParams(11, None)

    def computed_y(self) -> bool:
        return self.fixed_y is None


def aabft_sigma(n: int, mantissa_bits: int, y: float) -> float:
    """aabft_sigma (threshold_aabft.cpp:31-36)."""
    out = C.c_double()
    check(lib.vabft_aabft_sigma(int(n), int(mantissa_bits), float(y), C.byref(out)))
    return out.value


@dataclass
class AabftThresholds:
    per_row: np.ndarray
    y_used: float = 0.0
    degenerate: bool = False


def aabft_threshold(a: np.ndarray, b: np.ndarray, params: AabftParams, spec="fp64") -> AabftThresholds:
    """aabft_threshold (threshold_aabft.cpp:50-60) on the GPU, n = K."""
    s = _spec(spec)
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape[1] != b.shape[0]:
        raise _capi.InvalidArgument("aabft_threshold: inner dimensions disagree")
    m, k = a.shape
    n = b.shape[1]
    dA, dB = to_device(a, s.format), to_device(b, s.format)
    T = torch.empty(m, dtype=torch.float64, device="cuda")
    y = C.c_double()
    dg = C.c_int32()
    # NaN = computed y (AabftParams::fixed_y empty); any other value, zero
    # included, is a fixed y as in the reference
    fixed = math.nan if params.fixed_y is None else float(params.fixed_y)
    check(lib.vabft_aabft_threshold(s.code, m, n, k, ptr(dA), ptr(dB), params.mantissa_bits, fixed,
                                    params.confidence_multiplier, ptr(T), C.byref(y), C.byref(dg), stream_ptr()))
    torch.cuda.synchronize()
    return AabftThresholds(to_host(T), y.value, bool(dg.value))


def aabft_computed_y(a: np.ndarray, b: np.ndarray, spec="fp64") -> float:
    """aabft_computed_y (threshold_aabft.cpp:38-48)."""
    return aabft_threshold(a, b, AabftParams(53, None), spec).y_used


# ---------------------------------------------------------------- detect
@dataclass
class RowVerdict:
    """vabft::RowVerdict (detect.hpp:14-23)."""
    row: int = 0
    diff1: float = 0.0
    diff2: float = 0.0
    threshold: float = 0.0
    detected: bool = False
    location: Optional[int] = None
    correction: Optional[float] = None
    localization_residual: float = 0.0


@dataclass
class DetectOptions:
    localization_floor_scale: float = 1e-3
    residual_margin: float = 0.1


def localize(d1: float, d2: float, n_cols: int):
    """localize (detect.cpp:9-17): (j, residual) or None."""
    j = C.c_int64()
    r = C.c_double()
    ok = lib.vabft_localize(float(d1), float(d2), int(n_cols), C.byref(j), C.byref(r))
    return (j.value, r.value) if ok else None


def verify_arrays(source: np.ndarray, src_format: str, row_check1, row_check2, thresholds,
                  checksum_precision: PrecisionSpec, opts: DetectOptions = DetectOptions()):
    """verify (detect.cpp:19-55) returning structure-of-arrays verdicts."""
    source = np.asarray(source, dtype=np.float64)
    m, n = source.shape
    th = np.asarray(thresholds, dtype=np.float64)
    if th.shape != (m,):
        raise _capi.InvalidArgument("verify: thresholds length must equal row count")
    dS = to_device(source, src_format)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()  # noqa: E731
    rc1, rc2, T = t(row_check1), t(row_check2), t(th)
    d1, d2, res = (torch.empty(m, dtype=torch.float64, device="cuda") for _ in range(3))
    det = torch.empty(m, dtype=torch.uint8, device="cuda")
    loc = torch.empty(m, dtype=torch.int64, device="cuda")
    counts = torch.zeros(_capi.NUM_COUNTS, dtype=torch.int64, device="cuda")
    v = _capi.Verdicts(ptr(d1), ptr(d2), ptr(det), ptr(loc), ptr(res), None, None)
    check(lib.vabft_verify(C.byref(checksum_precision.to_c()), _capi.FORMAT_CODES[src_format], m, n, ptr(dS),
                           ptr(rc1), ptr(rc2), ptr(T), opts.localization_floor_scale, v, ptr(counts),
                           stream_ptr()))
    torch.cuda.synchronize()
    return {"diff1": to_host(d1), "diff2": to_host(d2), "detected": det.cpu().numpy().astype(bool),
            "location": loc.cpu().numpy(), "residual": to_host(res), "counts": counts.cpu().numpy()}


def verify(prod: EncodedProduct, thresholds, opts: DetectOptions = DetectOptions()) -> list:
    """verify (detect.cpp:19-55): one RowVerdict per row."""
    th = np.asarray(thresholds, dtype=np.float64)
    if np.any(~(th >= 0.0)):
        raise _capi.InvalidArgument("verify: thresholds must be >= 0")
    r = verify_arrays(prod.verification_source(), prod.verification_format(), prod.row_check1,
                      prod.row_check2, th, prod.checksum_precision, opts)
    out = []
    for i in range(th.size):
        loc = int(r["location"][i])
        out.append(RowVerdict(i, float(r["diff1"][i]), float(r["diff2"][i]), float(th[i]), bool(r["detected"][i]),
                              loc if loc >= 0 else None, float(r["diff1"][i]) if loc >= 0 else None,
                              float(r["residual"][i])))
    return out


def correct(c: np.ndarray, verdict: RowVerdict, spec) -> np.ndarray:
    """correct (detect.cpp:57-64): C[row][loc] = quantize(C - correction)."""
    if not verdict.detected or verdict.location is None or verdict.correction is None:
        raise _capi.InvalidArgument("correct: verdict has no usable location")
    out = np.array(c, dtype=np.float64, copy=True)
    i, j = verdict.row, verdict.location
    out[i, j] = quantize(c[i, j] - verdict.correction, spec)
    return out


# ---------------------------------------------------------------- faults
def encode_bits(value: float, fmt) -> int:
    """encode_bits (faults.cpp:66-76)."""
    out = C.c_uint64()
    check(lib.vabft_encode_bits(float(value), _capi.FORMAT_CODES[fmt_name(fmt)], C.byref(out)))
    return out.value


def decode_bits(bits: int, fmt) -> float:
    """decode_bits (faults.cpp:78-87)."""
    out = C.c_double()
    check(lib.vabft_decode_bits(int(bits), _capi.FORMAT_CODES[fmt_name(fmt)], C.byref(out)))
    return out.value


@dataclass
class FaultSpec:
    """vabft::FaultSpec (faults.hpp:21-26) with a fixed position."""
    position: tuple
    bit_index: int = 0
    direction: int = FlipDirection.FLIP


@dataclass
class InjectionRecord:
    i: int = -1
    j: int = -1
    bit: int = 0
    direction_taken: int = FlipDirection.FLIP
    value_before: float = 0.0
    value_after: float = 0.0
    applied: bool = False


def inject(m: np.ndarray, spec, fault: FaultSpec):
    """inject (faults.cpp:104-168) at a fixed position, executed on the GPU.
    Returns (matrix copy, InjectionRecord)."""
    fmt = _spec(spec).format if not isinstance(spec, str) else spec
    if fault.direction == FlipDirection.ANY:
        raise _capi.InvalidArgument("inject: direction ANY needs an RNG draw; resolve it first")
    m = np.asarray(m, dtype=np.float64)
    d = to_device(m, fmt)
    f = _capi.Fault(int(fault.position[0]), int(fault.position[1]), int(fault.bit_index), int(fault.direction))
    rec = _capi.FaultRecord()
    check(lib.vabft_inject(_capi.FORMAT_CODES[fmt], m.shape[0], m.shape[1], ptr(d), C.byref(f), 1, C.byref(rec),
                           stream_ptr()))
    out = to_host(d)
    r = InjectionRecord(f.i, f.j, f.bit, f.direction, rec.value_before, rec.value_after, bool(rec.applied))
    return out, r
