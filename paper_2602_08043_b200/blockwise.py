"""Block-wise (tile-level) V-ABFT (PAPER.md §"Integration with Block-wise
ABFT"): statistics per block of A and B, the V-ABFT formula
per block, block checksums aggregated for the verification.

Tiles (tile_k, tile_n) (the paper's (M, K, N) = (128, 1024, 256)):
  * column blocks J of tile_n columns are independent ABFT units — row
    checksums A (B_J r) against the row sums of C[:, J], position weights
    local to J, location = local column + J's offset (the N-slice semantics
    of sharding.shard_columns);
  * k-tiles of tile_k contribute their own bound: T_iJ = sum over k-tiles kt
    of vabft_threshold(A[i, kt] stats, B[kt, J] stats, n = |J|, e_max(|kt|))
    — the per-tile rounding errors add up in the accumulated C.
Every piece is the reference's own function on a slice (vabft_thresholds,
encode_and_multiply, verify — threshold_vabft.cpp:54-61, checksum.cpp:150-158,
detect.cpp:19-55), run on the device, so each block is exactly as
reproducible as the full-row path.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import numpy as np
import torch

from . import _capi, api
from ._capi import check, lib
from .device import ptr, stream_ptr, to_device, to_host


@dataclass
class BlockVerdicts:
    detected: np.ndarray   # [M] bool: any block of the row flagged
    location: np.ndarray   # [M] int64: global column of the first flagged block's location, -1 if none
    block_detected: np.ndarray  # [M, nJ] bool
    diff1: np.ndarray      # [M, nJ]
    thresholds: np.ndarray  # [M, nJ]
    col_blocks: List[tuple]


def col_blocks(n: int, tile_n: int) -> List[tuple]:
    return [(j0, min(j0 + tile_n, n)) for j0 in range(0, n, tile_n)]


def k_tiles(k: int, tile_k: int) -> List[tuple]:
    return [(k0, min(k0 + tile_k, k)) for k0 in range(0, k, tile_k)]


def _tile_emax(fmt: str, k: int, tile_k: int, e_max: Optional[float]) -> np.ndarray:
    return np.array([e_max if e_max is not None else api.resolve_e_max(fmt, k1 - k0) for (k0, k1) in k_tiles(k, tile_k)],
                    dtype=np.float64)


def blockwise_thresholds_device(A: torch.Tensor, B: torch.Tensor, fmt: str, tile_k: int = 1024, tile_n: int = 256,
                                e_max: Optional[float] = None, c_sigma: float = 2.5) -> torch.Tensor:
    """T[i, J] for CUDA operands in their storage format (bf16 / fp16 / fp32 /
    fp64 tensors, row strides honoured): one C-ABI call, three launches
    (csrc/blockwise.cu) — segment row statistics, the per-(k-tile, block)
    B summaries as independent chains, the k-tile sums. Returns an M x nJ
    float64 CUDA tensor."""
    m, k = A.shape
    n = B.shape[1]
    if B.shape[0] != k:
        raise _capi.InvalidArgument("blockwise_thresholds: inner dimensions disagree")
    if A.stride(1) != 1 or B.stride(1) != 1:
        raise _capi.InvalidArgument("blockwise_thresholds: rows must be contiguous")
    em = _tile_emax(fmt, k, tile_k, e_max)
    T = torch.empty(m, (n + tile_n - 1) // tile_n, dtype=torch.float64, device=A.device)
    check(lib.vabft_blockwise_thresholds(api._spec(fmt).code, m, n, k, ptr(A), A.stride(0), ptr(B), B.stride(0),
                                         tile_k, tile_n, em.ctypes.data, c_sigma, ptr(T), stream_ptr()))
    return T


def blockwise_thresholds(a: np.ndarray, b: np.ndarray, fmt: str, tile_k: int = 1024, tile_n: int = 256,
                         e_max: Optional[float] = None, c_sigma: float = 2.5, engine: str = "device") -> np.ndarray:
    """T[i, J] = sum_kt vabft_threshold(A[i, kt], B[kt, J], n = |J|), with
    e_max per k-tile from the format model at dim = |kt| unless given.
    engine "device": one call of the block-wise kernels; "slices": the
    composition slice pair by slice pair through vabft_thresholds (the
    reference's own function on each slice — the check of the kernels)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if engine == "device":
        s = api._spec(fmt)
        return to_host(blockwise_thresholds_device(to_device(a, s.format), to_device(b, s.format), fmt, tile_k,
                                                   tile_n, e_max, c_sigma))
    m, k = a.shape
    blocks = col_blocks(b.shape[1], tile_n)
    T = np.zeros((m, len(blocks)))
    for (k0, k1) in k_tiles(k, tile_k):
        e = e_max if e_max is not None else api.resolve_e_max(fmt, k1 - k0)
        a_kt = np.ascontiguousarray(a[:, k0:k1])
        for jb, (j0, j1) in enumerate(blocks):
            T[:, jb] += api.vabft_thresholds(a_kt, np.ascontiguousarray(b[k0:k1, j0:j1]),
                                             api.VabftParams(e, c_sigma), fmt)
    return T


def blockwise_verify(a: np.ndarray, b: np.ndarray, c: Optional[np.ndarray], fmt: str, mode: str = "offline",
                     tile_k: int = 1024, tile_n: int = 256, e_max: Optional[float] = None, c_sigma: float = 2.5,
                     engine: str = "exact") -> BlockVerdicts:
    """Verify C (or the product itself when c is None) block by block."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m = a.shape[0]
    blocks = col_blocks(b.shape[1], tile_n)
    T = blockwise_thresholds(a, b, fmt, tile_k, tile_n, e_max, c_sigma)
    det = np.zeros((m, len(blocks)), dtype=bool)
    d1 = np.zeros((m, len(blocks)))
    loc = np.full(m, -1, dtype=np.int64)
    for jb, (j0, j1) in enumerate(blocks):
        prod = api.encode_and_multiply(a, np.ascontiguousarray(b[:, j0:j1]), mode, fmt, engine=engine)
        if c is not None:
            cj = np.ascontiguousarray(np.asarray(c, dtype=np.float64)[:, j0:j1])
            prod.c = cj
            prod.c_accum = cj
        v = api.verify_arrays(prod.verification_source(), prod.verification_format(), prod.row_check1,
                              prod.row_check2, T[:, jb], prod.checksum_precision)
        det[:, jb] = v["detected"]
        d1[:, jb] = v["diff1"]
        first = (loc < 0) & v["detected"] & (v["location"] >= 0)
        loc[first] = v["location"][first] + j0
    return BlockVerdicts(det.any(axis=1), loc, det, d1, T, blocks)
