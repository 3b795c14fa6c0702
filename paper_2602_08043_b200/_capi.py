"""ctypes binding of the C-ABI in include/vabft_c.h (libvabft_b200.so).

The shared library is built in-tree (``make -C paper_2602_08043_b200/csrc``).
There is no CPU fallback: importing this module without the library raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvabft_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first "
        "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")

lib = C.CDLL(LIB_PATH)

# enums -----------------------------------------------------------------
OK, INVALID_ARGUMENT, DOMAIN_ERROR, RANGE_ERROR, OUT_OF_RANGE, LOGIC_ERROR, CUDA_ERROR, UNSUPPORTED = range(8)
BF16, FP16, FP32, FP64 = range(4)
ACCUM_FP32_ROUND_OUTPUT, ACCUM_SEQUENTIAL, ACCUM_BLOCKED, ACCUM_PAIRWISE = range(4)
OFFLINE, ONLINE = 0, 1
FLIP, SET0TO1, SET1TO0, ANY = range(4)
ENGINE_EXACT, ENGINE_TENSOR = 0, 1
COUNT_ROWS, COUNT_DETECTED, COUNT_LOCATED, COUNT_NAN, COUNT_SLOW_STATS, COUNT_CORRECTED, NUM_COUNTS = \
    0, 1, 2, 3, 4, 5, 6

FORMAT_CODES = {"bf16": BF16, "fp16": FP16, "fp32": FP32, "fp64": FP64}


class Accum(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("block_len", C.c_int64)]


class Precision(C.Structure):
    _fields_ = [("format", C.c_int32), ("mantissa_bits", C.c_int32), ("unit_roundoff", C.c_double),
                ("accumulation", Accum), ("emax_kind", C.c_int32), ("overflow", C.c_int32),
                ("emax_scale", C.c_double), ("emax_offset", C.c_double)]


class Verdicts(C.Structure):
    _fields_ = [("diff1", C.c_void_p), ("diff2", C.c_void_p), ("detected", C.c_void_p),
                ("location", C.c_void_p), ("residual", C.c_void_p), ("row_check1", C.c_void_p),
                ("row_check2", C.c_void_p)]


class Fault(C.Structure):
    _fields_ = [("i", C.c_int64), ("j", C.c_int64), ("bit", C.c_int32), ("direction", C.c_int32)]


class FaultRecord(C.Structure):
    _fields_ = [("value_before", C.c_double), ("value_after", C.c_double), ("applied", C.c_int32),
                ("reserved", C.c_int32)]


class FusedOpts(C.Structure):
    _fields_ = [("mode", C.c_int32), ("threshold_method", C.c_int32), ("e_max", C.c_double),
                ("c_sigma", C.c_double), ("floor_scale", C.c_double), ("aabft_mantissa_bits", C.c_int32),
                ("b_kmajor", C.c_int32), ("aabft_fixed_y", C.c_double), ("aabft_confidence", C.c_double),
                ("fault_col", C.c_void_p), ("fault_bit", C.c_void_p), ("fault_dir", C.c_void_p),
                ("fault_records", C.c_void_p), ("stages", C.c_int32), ("fault_target", C.c_int32),
                ("n_operand_faults", C.c_int32), ("correct", C.c_int32), ("operand_faults", C.c_void_p),
                ("operand_fault_records", C.c_void_p), ("cta_mode", C.c_int32), ("tf32_passes", C.c_int32),
                ("accum_out", C.c_void_p), ("workspace_fresh", C.c_int32), ("reserved_v2", C.c_int32),
                ("lda", C.c_int64), ("ldc", C.c_int64), ("t_in", C.c_void_p), ("ldt", C.c_int64)]


_st = C.c_int
_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_d = C.c_double
_dp = C.POINTER(C.c_double)

_SIGS = {
    "vabft_last_error": (C.c_char_p, []),
    "vabft_api_version": (C.c_int32, []),
    "vabft_precision_default": (_st, [_i32, C.POINTER(Precision)]),
    "vabft_quantize": (_st, [_d, C.POINTER(Precision), _dp]),
    "vabft_resolve_e_max": (_st, [C.POINTER(Precision), _i64, _dp]),
    "vabft_aabft_sigma": (_st, [_i64, _i32, _d, _dp]),
    "vabft_threshold_row": (_st, [_dp, _dp, _i64, _d, _d, _dp]),
    "vabft_localize": (C.c_int32, [_d, _d, _i64, C.POINTER(C.c_int64), _dp]),
    "vabft_encode_bits": (_st, [_d, _i32, C.POINTER(C.c_uint64)]),
    "vabft_decode_bits": (_st, [C.c_uint64, _i32, _dp]),
    "vabft_device_info": (_st, [C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "vabft_encode_workspace_size": (_st, [_i64, _i64, _i64, C.POINTER(Precision), C.POINTER(C.c_size_t)]),
    "vabft_encode_and_multiply": (_st, [C.POINTER(Precision), _i32, _i32, _i64, _i64, _i64, _vp, _vp, _vp, _vp,
                                        _vp, _vp, _vp, _vp, _vp, C.c_size_t, _vp]),
    "vabft_row_sums": (_st, [C.POINTER(Precision), _i32, _i64, _i64, _vp, _vp, _vp, _vp]),
    "vabft_row_stats": (_st, [_i32, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "vabft_vabft_thresholds": (_st, [_i32, _i64, _i64, _i64, _vp, _vp, _d, _d, _vp, _vp, _vp]),
    "vabft_blockwise_thresholds": (_st, [_i32, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _vp, _d, _vp,
                                         _vp]),
    "vabft_aabft_threshold": (_st, [_i32, _i64, _i64, _i64, _vp, _vp, _i32, _d, _d, _vp, _dp,
                                    C.POINTER(C.c_int32), _vp]),
    "vabft_verify": (_st, [C.POINTER(Precision), _i32, _i64, _i64, _vp, _vp, _vp, _vp, _d, Verdicts, _vp, _vp]),
    "vabft_inject": (_st, [_i32, _i64, _i64, _vp, C.POINTER(Fault), _i64, C.POINTER(FaultRecord), _vp]),
    "vabft_bside_create": (_st, [_i32, _i32, _i64, _i64, _vp, C.POINTER(_vp), _vp]),
    "vabft_bside_create_ld": (_st, [_i32, _i32, _i64, _i64, _vp, _i64, C.POINTER(_vp), _vp]),
    "vabft_bside_update": (_st, [_vp, _vp, _vp]),
    "vabft_bside_destroy": (_st, [_vp]),
    "vabft_fused_workspace_size": (_st, [_i64, _i64, _i64, C.POINTER(C.c_size_t)]),
    "vabft_fused_gemm": (_st, [C.POINTER(FusedOpts), _vp, _i64, _vp, _vp, _vp, Verdicts, _vp, _vp, C.c_size_t, _vp]),
    "vabft_gemm_plain": (_st, [_i32, _i32, _i64, _i64, _i64, _vp, _vp, _vp, _vp]),
    "vabft_gemm_plain_mode": (_st, [_i32, _i32, _i64, _i64, _i64, _vp, _vp, _vp, _i32, _vp]),
    "vabft_fused_uses_cta_pairs": (_i32, [C.POINTER(FusedOpts), _i64, _i64, _i64]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIGS)


class VabftError(RuntimeError):
    """Base of the C-ABI errors; subclasses mirror the reference's exception types."""


class InvalidArgument(VabftError, ValueError):
    pass


class DomainError(VabftError, ValueError):
    pass


class RangeError(VabftError, ArithmeticError):
    pass


class OutOfRange(VabftError, IndexError):
    pass


class LogicError(VabftError):
    pass


class CudaError(VabftError):
    pass


class Unsupported(VabftError):
    pass


_ERRORS = {INVALID_ARGUMENT: InvalidArgument, DOMAIN_ERROR: DomainError, RANGE_ERROR: RangeError,
           OUT_OF_RANGE: OutOfRange, LOGIC_ERROR: LogicError, CUDA_ERROR: CudaError, UNSUPPORTED: Unsupported}


def check(status: int) -> None:
    if status != OK:
        msg = lib.vabft_last_error().decode()
        raise _ERRORS.get(status, VabftError)(msg)


def precision(fmt) -> Precision:
    p = Precision()
    check(lib.vabft_precision_default(FORMAT_CODES.get(fmt, fmt), C.byref(p)))
    return p
