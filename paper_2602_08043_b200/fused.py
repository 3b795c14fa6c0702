"""The hot path on device tensors: the tcgen05 fused V-ABFT GEMM.

    g = FusedAbftGemm(B, mode="online")          # per-weight B-side state
    r = g(A)                                     # C, thresholds, verdicts, counts

One call = A-side statistics (row stats -> V-ABFT thresholds, A (B r)
checksums), the tcgen05 GEMM with the ABFT epilogue, and the verify tail —
all stream-ordered on the current torch stream, no host synchronization.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import torch

from . import _capi
from ._capi import check, lib
from .emax import default_e_max
from .device import ptr, stream_ptr

_FMT = {torch.bfloat16: _capi.BF16, torch.float16: _capi.FP16, torch.float32: _capi.FP32,
        torch.float64: _capi.FP64}
_METHOD = {"vabft": 0, "aabft-fixed-y": 1, "aabft-computed-y": 2}
_TARGET = {"output": 0, "A": 1, "B": 2}  # FaultTarget (faults.hpp:15)


def operand_faults(faults, device="cuda") -> torch.Tensor:
    """vabft_fault array for B-operand faults: [(k, j, bit, direction), ...]
    -> an int64 [n, 3] device tensor with the C struct layout
    {int64 i = k, int64 j, int32 bit, int32 direction}."""
    rows = [[int(k), int(j), (int(bit) & 0xFFFFFFFF) | (int(d) << 32)] for (k, j, bit, d) in faults]
    return torch.tensor(rows, dtype=torch.int64, device=device).reshape(-1, 3)

_FMT_NAME = {torch.bfloat16: "bf16", torch.float16: "fp16", torch.float32: "fp32", torch.float64: "fp64"}


@dataclass
class FusedResult:
    C: torch.Tensor
    T: Optional[torch.Tensor]
    diff1: Optional[torch.Tensor]
    diff2: Optional[torch.Tensor]
    detected: Optional[torch.Tensor]
    location: Optional[torch.Tensor]
    residual: Optional[torch.Tensor]
    counts: Optional[torch.Tensor]
    row_check1: Optional[torch.Tensor] = None
    row_check2: Optional[torch.Tensor] = None


class FusedAbftGemm:
    """Fault-tolerant C = A B for a fixed weight B (K x N, row-major): BF16 /
    FP16 on the tcgen05 kernel, FP32 on tcgen05 kind::tf32 (3xTF32, or one
    TF32 pass with tf32_passes=1), FP64 on the SIMT DFMA kernel (K5)."""

    def __init__(self, B: torch.Tensor, mode: str = "online", threshold: str = "vabft",
                 e_max: Optional[float] = None, c_sigma: float = 2.5, floor_scale: float = 1e-3,
                 aabft_mantissa_bits: int = 0, aabft_fixed_y: float = 21.0, aabft_confidence: float = 3.0,
                 tf32_passes: int = 3):
        if B.dtype not in _FMT or not B.is_cuda or B.dim() != 2:
            raise _capi.InvalidArgument("FusedAbftGemm: B must be a 2-D BF16/FP16/FP32/FP64 CUDA tensor")
        # a row-strided view (e.g. a column slice B[:, n0:n1] of a wider
        # weight) is used in place for BF16 / FP16 (row stride a multiple of 8)
        strided_ok = B.dtype in (torch.bfloat16, torch.float16) and B.stride(1) == 1 and B.stride(0) % 8 == 0
        self.B = B if (B.is_contiguous() or strided_ok) else B.contiguous()
        self.ldb = self.B.stride(0)
        self.fmt = _FMT[B.dtype]
        self.k, self.n = self.B.shape
        self.mode = _capi.ONLINE if mode == "online" else _capi.OFFLINE
        if e_max is None:
            # resolve_run_e_max (harness.cpp): the calibrated model at dim = K
            name = "tf32" if (B.dtype == torch.float32 and tf32_passes == 1) else _FMT_NAME[B.dtype]
            e_max = default_e_max(name, "online" if self.mode == _capi.ONLINE else "offline", self.k)
        self.opts = _capi.FusedOpts()
        self.opts.mode = self.mode
        self.opts.threshold_method = _METHOD[threshold]
        self.opts.e_max = e_max
        self.opts.c_sigma = c_sigma
        self.opts.floor_scale = floor_scale
        self.opts.aabft_mantissa_bits = aabft_mantissa_bits
        self.opts.b_kmajor = 0
        self.opts.aabft_fixed_y = aabft_fixed_y
        self.opts.aabft_confidence = aabft_confidence
        self.opts.cta_mode = -1
        self.opts.tf32_passes = tf32_passes  # FP32 weights: 3xTF32 (default) or one TF32 pass
        self.h = C.c_void_p()
        check(lib.vabft_bside_create_ld(self.fmt, self.mode, self.k, self.n, ptr(self.B), self.ldb, C.byref(self.h),
                                        stream_ptr()))
        self._ws = None
        self._bufs = {}

    def uses_cta_pairs(self, m: int) -> bool:
        """Whether a launch of M rows runs the CTA-pair (cta_group::2) kernel."""
        return bool(lib.vabft_fused_uses_cta_pairs(C.byref(self.opts), m, self.n, self.k))

    def update_weight(self, B: torch.Tensor) -> None:
        if tuple(B.shape) != (self.k, self.n) or B.stride() != self.B.stride():
            raise _capi.InvalidArgument("update_weight: same shape and strides as the handle's weight")
        self.B = B
        check(lib.vabft_bside_update(self.h, ptr(self.B), stream_ptr()))

    def workspace(self, m: int) -> torch.Tensor:
        sz = C.c_size_t()
        check(lib.vabft_fused_workspace_size(m, self.n, self.k, C.byref(sz)))
        if self._ws is None or self._ws.numel() < sz.value:
            self._ws = torch.empty(sz.value, dtype=torch.uint8, device=self.B.device)
        return self._ws

    def __call__(self, A: torch.Tensor, out: Optional[torch.Tensor] = None, *, verdicts: bool = True,
                 thresholds: bool = True, counts: Optional[torch.Tensor] = None,
                 faults: Optional[dict] = None, stages: int = 0, checksums: bool = False,
                 correct: bool = False, accum_out: Optional[torch.Tensor] = None,
                 t_in: Optional[torch.Tensor] = None) -> FusedResult:
        """faults: {"target": "output" | "A" | "B", ...}. output / A: per-row
        int32 tensors "col" (output column, or the k index of A[i][k]; < 0 =
        none), "bit", "dir" and optional "records" (M x 24-byte records). B:
        "operand" = operand_faults(...) and optional "records" (per fault).
        correct: in-kernel correction of located single errors.
        accum_out: M x N FP32 tensor receiving the (post-injection) FP32
        accumulator that online verification reads (BF16 / FP16 weights).
        t_in: given thresholds (threshold method 3) — a float64 CUDA vector of
        M values, any stride (e.g. a column of blockwise_thresholds_device)."""
        if A.dtype != self.B.dtype or A.dim() != 2 or A.shape[1] != self.k:
            raise _capi.InvalidArgument("FusedAbftGemm: A must be M x K with B's dtype")
        m = A.shape[0]
        sixteen = A.dtype in (torch.bfloat16, torch.float16)
        if not (sixteen and A.stride(1) == 1 and A.stride(0) % 8 == 0):
            A = A.contiguous()
        if out is not None and not (out.stride(1) == 1 and (out.is_contiguous() or (sixteen and out.stride(0) % 8 == 0))):
            raise _capi.InvalidArgument("FusedAbftGemm: out must be contiguous (BF16/FP16: or row-strided by a multiple of 8)")
        # output buffers are cached per M (valid until the next call with the
        # same M) so the hot loop allocates nothing
        bufs = self._bufs.get(m)
        if bufs is None:
            dev = A.device
            bufs = {"T": torch.empty(m, dtype=torch.float64, device=dev),
                    "d1": torch.empty(m, dtype=torch.float64, device=dev),
                    "d2": torch.empty(m, dtype=torch.float64, device=dev),
                    "res": torch.empty(m, dtype=torch.float64, device=dev),
                    "det": torch.empty(m, dtype=torch.uint8, device=dev),
                    "loc": torch.empty(m, dtype=torch.int64, device=dev),
                    "rc1": torch.empty(m, dtype=torch.float64, device=dev),
                    "rc2": torch.empty(m, dtype=torch.float64, device=dev)}
            self._bufs[m] = bufs
        if out is None and "C" not in bufs:  # only when the caller brings no output
            bufs["C"] = torch.empty((m, self.n), dtype=A.dtype, device=A.device)
        C_ = out if out is not None else bufs["C"]
        T = bufs["T"] if thresholds else None
        if verdicts:
            d1, d2, res, det, loc = bufs["d1"], bufs["d2"], bufs["res"], bufs["det"], bufs["loc"]
        else:
            d1 = d2 = res = det = loc = None
        rc1, rc2 = (bufs["rc1"], bufs["rc2"]) if checksums else (None, None)
        v = _capi.Verdicts(ptr(d1), ptr(d2), ptr(det), ptr(loc), ptr(res), ptr(rc1), ptr(rc2))
        opts = self.opts
        if stages:
            opts = _capi.FusedOpts.from_buffer_copy(self.opts)
            opts.stages = stages
        if faults is not None:
            opts = _capi.FusedOpts.from_buffer_copy(opts)
            target = faults.get("target", "output")
            opts.fault_target = _TARGET[target]
            if target == "B":
                op = faults["operand"]
                opts.operand_faults = ptr(op)
                opts.n_operand_faults = int(op.shape[0])
                opts.operand_fault_records = ptr(faults.get("records"))
            else:
                opts.fault_col = ptr(faults["col"])
                opts.fault_bit = ptr(faults["bit"])
                opts.fault_dir = ptr(faults["dir"])
                opts.fault_records = ptr(faults.get("records"))
        if correct:
            opts = _capi.FusedOpts.from_buffer_copy(opts)
            opts.correct = 1
        if accum_out is not None:
            if accum_out.dtype != torch.float32 or tuple(accum_out.shape) != (m, self.n) or not accum_out.is_contiguous():
                raise _capi.InvalidArgument("accum_out must be a contiguous M x N float32 tensor")
            opts = _capi.FusedOpts.from_buffer_copy(opts)
            opts.accum_out = ptr(accum_out)
        if t_in is not None:
            if t_in.dtype != torch.float64 or t_in.dim() != 1 or t_in.shape[0] != m or not t_in.is_cuda:
                raise _capi.InvalidArgument("t_in must be an M-vector of float64 on the device")
            opts = _capi.FusedOpts.from_buffer_copy(opts)
            opts.threshold_method = 3
            opts.t_in = ptr(t_in)
            opts.ldt = t_in.stride(0)
        if A.stride(0) != self.k or C_.stride(0) != self.n:
            opts = _capi.FusedOpts.from_buffer_copy(opts)
            opts.lda = A.stride(0)
            opts.ldc = C_.stride(0)
        ws = self.workspace(m)
        check(lib.vabft_fused_gemm(C.byref(opts), self.h, m, ptr(A), ptr(C_), ptr(T), v, ptr(counts),
                                   ptr(ws), ws.numel(), stream_ptr()))
        return FusedResult(C_, T, d1, d2, det, loc, res, counts, rc1, rc2)

    def close(self) -> None:
        if self.h:
            check(lib.vabft_bside_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def plain_gemm(A: torch.Tensor, B: torch.Tensor, out: Optional[torch.Tensor] = None, b_kmajor: bool = False,
               cta_mode: int = -1):
    """The same tcgen05 kernel with the ABFT epilogue compiled out (overhead
    baseline). cta_mode: -1 automatic (CTA pairs when eligible), 0 one CTA per
    128 x 256 tile, 1 CTA pairs (cta_group::2, 256 x 256)."""
    m, k = A.shape
    n = B.shape[0] if b_kmajor else B.shape[1]
    C_ = out if out is not None else torch.empty((m, n), dtype=A.dtype, device=A.device)
    check(lib.vabft_gemm_plain_mode(_FMT[A.dtype], int(b_kmajor), m, n, k, ptr(A), ptr(B), ptr(C_), int(cta_mode),
                                    stream_ptr()))
    return C_
