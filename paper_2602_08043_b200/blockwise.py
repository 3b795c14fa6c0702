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


def _tile_emax(fmt: str, k: int, tile_k: int, e_max) -> np.ndarray:
    """e_max per k-tile: given per tile (a sequence), one value for all, or
    the format model at dim = |kt| (resolve_e_max)."""
    tiles = k_tiles(k, tile_k)
    if e_max is not None and np.ndim(e_max) == 1:
        if len(e_max) != len(tiles):
            raise _capi.InvalidArgument("blockwise: one e_max per k-tile")
        return np.asarray(e_max, dtype=np.float64)
    return np.array([e_max if e_max is not None else api.resolve_e_max(fmt, k1 - k0) for (k0, k1) in tiles],
                    dtype=np.float64)


def blockwise_thresholds_device(A: torch.Tensor, B: torch.Tensor, fmt: str, tile_k: int = 1024, tile_n: int = 256,
                                e_max: Optional[float] = None, c_sigma: float = 2.5,
                                out: Optional[torch.Tensor] = None) -> torch.Tensor:
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
    nJ = (n + tile_n - 1) // tile_n
    T = out if out is not None else torch.empty(m, nJ, dtype=torch.float64, device=A.device)
    if tuple(T.shape) != (m, nJ) or T.dtype != torch.float64 or not T.is_contiguous():
        raise _capi.InvalidArgument("blockwise_thresholds: out must be a contiguous M x nJ float64 tensor")
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


@dataclass
class FusedBlockVerdicts:
    """Device tensors of blockwise_verify_fused (M x nJ unless noted)."""
    C: torch.Tensor            # M x N product
    thresholds: torch.Tensor   # float64
    block_detected: torch.Tensor  # uint8
    diff1: torch.Tensor        # float64
    location: torch.Tensor     # int64, global columns (-1: none)
    detected: torch.Tensor     # [M] bool: any block of the row flagged
    col_blocks: List[tuple]


class BlockwiseFusedGemm:
    """Block-wise V-ABFT on the fused path for one weight: per tile_n-column
    block J a fused handle over B[:, J] (a strided slice for BF16 / FP16 — no
    copy; the B-side statistics are per weight, built once), and per call the
    block-wise thresholds from the device kernels, then every block of C
    computed and verified by the fused tcgen05 kernel as its own ABFT unit
    (checksum weights local to J, as in the N-split) against T[:, J]
    (threshold method 3). Located columns are global."""

    def __init__(self, B: torch.Tensor, fmt: str, mode: str = "online", tile_k: int = 1024, tile_n: int = 256,
                 e_max=None, c_sigma: float = 2.5, graphs: bool = True, **fused_kw):
        from .fused import FusedAbftGemm
        self.use_graphs = graphs
        self._graphs = {}
        self.B, self.fmt, self.mode, self.tile_k, self.tile_n, self.c_sigma = B, fmt, mode, tile_k, tile_n, c_sigma
        k, n = B.shape
        if e_max is None:
            # the device calibration of the engine that accumulates (emax.py:
            # tcgen05 FP32 accumulation, 3xTF32 / one TF32 pass, DFMA) at each
            # k-tile's length — the reference's model is the emulator's
            from .emax import default_e_max
            name = "tf32" if (fmt == "fp32" and fused_kw.get("tf32_passes", 3) == 1) else fmt
            e_max = [default_e_max(name, mode, k1 - k0) for (k0, k1) in k_tiles(k, tile_k)]
        self.e_max = e_max
        self.blocks = col_blocks(n, tile_n)
        self.sixteen = B.dtype in (torch.bfloat16, torch.float16)
        # one stream per column block: a 256-column block's GEMM fills only
        # 2 x ceil(M / 256) SMs, so the blocks run side by side
        self.streams = [torch.cuda.Stream(device=B.device) for _ in self.blocks]
        self.handles = []
        for (j0, j1) in self.blocks:
            view = self.sixteen and j0 % 8 == 0 and (j1 - j0) % 8 == 0
            self.handles.append((FusedAbftGemm(B[:, j0:j1] if view else B[:, j0:j1].contiguous(), mode=mode,
                                               **fused_kw), view))

    def _blocks(self, A, T, Cm, det, d1, loc, cbs):
        """The column blocks on their streams (eager, or recorded into a graph)."""
        m = A.shape[0]
        main = torch.cuda.current_stream(A.device)
        for st in self.streams:
            st.wait_stream(main)  # T, the output buffers and the counters are ready
        for jb, ((j0, j1), (g, view)) in enumerate(zip(self.blocks, self.handles)):
            with torch.cuda.stream(self.streams[jb]):
                o = Cm[:, j0:j1] if view else torch.empty((m, j1 - j0), dtype=A.dtype, device=A.device)
                r = g(A, out=o, counts=cbs[jb] if cbs is not None else None, t_in=T[:, jb])
                if not view:
                    Cm[:, j0:j1] = o
                det[:, jb] = r.detected
                d1[:, jb] = r.diff1
                loc[:, jb] = torch.where(r.location >= 0, r.location + j0, r.location)
        for st in self.streams:
            main.wait_stream(st)

    def __call__(self, A: torch.Tensor, out: Optional[torch.Tensor] = None,
                 counts: Optional[torch.Tensor] = None) -> "FusedBlockVerdicts":
        """Block-wise verification of A B. With graphs on (the default) the
        16 per-block launches replay from a CUDA graph recorded per M (the
        eager per-block calls were host-bound): A is copied into the graph's
        input buffer, and C / the verdicts returned are the graph's buffers,
        valid until the next call with the same M (unless `out` is given)."""
        m = A.shape[0]
        n = self.B.shape[1]
        nJ = len(self.blocks)
        dev = A.device
        if self.use_graphs:
            st = self._graphs.get(m)
            if st is None:
                st = self._record(A)
            if st is not None:
                st["A"].copy_(A)
                blockwise_thresholds_device(st["A"], self.B, self.fmt, self.tile_k, self.tile_n, self.e_max,
                                            self.c_sigma, out=st["T"])
                st["graph"].replay()
                if counts is not None:
                    counts += st["cbs"].sum(dim=0)
                Cm = st["C"]
                if out is not None:
                    out.copy_(Cm)
                    Cm = out
                return self._verdicts(Cm, st["T"], st["det"], st["d1"], st["loc"], m, dev)
        T = blockwise_thresholds_device(A, self.B, self.fmt, self.tile_k, self.tile_n, self.e_max, self.c_sigma)
        Cm = out if out is not None else torch.empty((m, n), dtype=A.dtype, device=dev)
        det = torch.empty((m, nJ), dtype=torch.uint8, device=dev)
        d1 = torch.empty((m, nJ), dtype=torch.float64, device=dev)
        loc = torch.empty((m, nJ), dtype=torch.int64, device=dev)
        cbs = torch.zeros((nJ, 6), dtype=torch.int64, device=dev) if counts is not None else None
        self._blocks(A, T, Cm, det, d1, loc, cbs)
        if counts is not None:
            counts += cbs.sum(dim=0)
        return self._verdicts(Cm, T, det, d1, loc, m, dev)

    def _record(self, A):
        m, k = A.shape
        n = self.B.shape[1]
        nJ = len(self.blocks)
        dev = A.device
        st = {"A": torch.empty_like(A, memory_format=torch.contiguous_format),
              "T": torch.empty((m, nJ), dtype=torch.float64, device=dev),
              "C": torch.empty((m, n), dtype=A.dtype, device=dev),
              "det": torch.empty((m, nJ), dtype=torch.uint8, device=dev),
              "d1": torch.empty((m, nJ), dtype=torch.float64, device=dev),
              "loc": torch.empty((m, nJ), dtype=torch.int64, device=dev),
              "cbs": torch.zeros((nJ, 6), dtype=torch.int64, device=dev)}
        st["A"].copy_(A)
        blockwise_thresholds_device(st["A"], self.B, self.fmt, self.tile_k, self.tile_n, self.e_max, self.c_sigma,
                                    out=st["T"])
        args = (st["A"], st["T"], st["C"], st["det"], st["d1"], st["loc"], st["cbs"])
        try:
            self._blocks(*args)  # eager once: handles' buffers and workspaces exist before recording
            torch.cuda.synchronize(dev)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                st["cbs"].zero_()
                self._blocks(*args)
            st["graph"] = g
        except Exception:
            self.use_graphs = False
            return None
        self._graphs[m] = st
        return st

    def _verdicts(self, Cm, T, det, d1, loc, m, dev) -> "FusedBlockVerdicts":
        flagged = det.bool()
        # the first flagged block with a located column (blockwise_verify's rule)
        hit = flagged & (loc >= 0)
        first = hit.int().argmax(dim=1)
        location = torch.where(hit.any(dim=1), loc.gather(1, first[:, None])[:, 0],
                               torch.full((m,), -1, dtype=torch.int64, device=dev))
        return FusedBlockVerdicts(Cm, T, det, d1, location, flagged.any(dim=1), self.blocks)

    def close(self) -> None:
        self._graphs = {}
        for g, _ in self.handles:
            g.close()
        self.handles = []


def blockwise_verify_fused(A: torch.Tensor, B: torch.Tensor, fmt: str, mode: str = "online", tile_k: int = 1024,
                           tile_n: int = 256, e_max=None, c_sigma: float = 2.5,
                           counts: Optional[torch.Tensor] = None, **fused_kw) -> FusedBlockVerdicts:
    """One-shot BlockwiseFusedGemm (handles built and released per call)."""
    g = BlockwiseFusedGemm(B, fmt, mode, tile_k, tile_n, e_max, c_sigma, graphs=False, **fused_kw)
    try:
        return g(A, counts=counts)
    finally:
        g.close()
