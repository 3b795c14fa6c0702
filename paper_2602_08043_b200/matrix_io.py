"""Matrix files and verify_files — the data formats and the file-driven caller
around the hot path.

  VABFTMAT binary   magic "VABFTMAT", u32 version (1), u8 format id, u64 rows,
                    u64 cols, then rows*cols little-endian FP64 values
                    (matrix_io.hpp:12-17, matrix_io.cpp:49-88)
  CSV               one matrix row per line, comma separated, %.17g
                    (matrix_io.cpp:90-125)
  load_matrix_auto  binary by magic, else CSV in the given format
                    (matrix_io.cpp:127-137)

Loading quantizes finite values onto the format's grid (Matrix::set) and keeps
non-finite values raw (fill_values, matrix_io.cpp:34-45), so corrupted products
round-trip. verify_files (harness.cpp:430-490) then runs the hot path on the
GPU: encode_and_multiply, vabft_thresholds, verify — against the product
itself or an external C (`check_against`) — and returns the reference's JSON
document and exit code (2 if any row is flagged, else 0).

File I/O is host work; every numeric step after loading runs on the device.
"""
from __future__ import annotations

import math
import os
import struct
import time
from typing import Optional, Tuple

import numpy as np

from . import _capi, api

MAGIC = b"VABFTMAT"
VERSION = 1
FORMATS = ("bf16", "fp16", "fp32", "fp64")
_HEADER = struct.Struct("<8sIBQQ")  # magic, version, format id, rows, cols (packed: 29 bytes)

# (t = significand bits incl. the implicit one, emin, max finite) per format
_GRID = {"bf16": (8, -126, float.fromhex("0x1.FEp127")), "fp16": (11, -14, 65504.0),
         "fp32": (24, -126, float(np.finfo(np.float32).max)), "fp64": (53, -1022, float(np.finfo(np.float64).max))}


class MatrixFileError(RuntimeError):
    """std::runtime_error of matrix_io.cpp."""


def quantize_array(x: np.ndarray, fmt: str) -> np.ndarray:
    """quantize (precision.cpp:129-159) element-wise for finite values with the
    Saturate policy: RNE to t bits, subnormals kept (quantum of the format's
    minimum exponent), |y| > max finite -> +-max finite. Non-finite values
    pass through (fill_values keeps them raw)."""
    x = np.asarray(x, dtype=np.float64)
    if fmt == "fp64":
        return x.copy()
    t, emin, mx = _GRID[fmt]
    out = x.copy()
    fin = np.isfinite(x) & (x != 0.0)
    v = x[fin]
    _, e = np.frexp(v)  # v = m 2^e, 0.5 <= |m| < 1 -> unbiased exponent e - 1
    q = np.ldexp(1.0, np.maximum(e - 1, emin) - (t - 1))  # quantum
    y = np.rint(v / q) * q  # exact scaling by a power of two; rint = ties to even
    y = np.where(np.abs(y) > mx, np.copysign(mx, y), y)
    out[fin] = y
    return out


def save_matrix_binary(values: np.ndarray, fmt: str, path: str) -> None:
    """save_matrix_binary (matrix_io.cpp:49-60)."""
    v = np.ascontiguousarray(values, dtype="<f8")
    if v.ndim != 2:
        raise _capi.InvalidArgument("save_matrix_binary: a 2-D matrix is required")
    try:
        with open(path, "wb") as f:
            f.write(_HEADER.pack(MAGIC, VERSION, FORMATS.index(fmt), v.shape[0], v.shape[1]))
            f.write(v.tobytes())
    except OSError as e:
        raise MatrixFileError(f"cannot open for writing: {path}") from e


def load_matrix_binary(path: str) -> Tuple[np.ndarray, str]:
    """load_matrix_binary (matrix_io.cpp:62-88): (values, format)."""
    try:
        with open(path, "rb") as f:
            head = f.read(_HEADER.size)
            if len(head) < 8 or head[:8] != MAGIC:
                raise MatrixFileError(f"not a VABFTMAT file: {path}")
            if len(head) < _HEADER.size:
                raise MatrixFileError(f"truncated matrix file: {path}")
            _, version, fmt_id, rows, cols = _HEADER.unpack(head)
            if version != VERSION:
                raise MatrixFileError(f"unsupported matrix file version in {path}")
            if fmt_id > 3:
                raise MatrixFileError(f"bad format id in {path}")
            if rows < 1 or cols < 1 or rows > (1 << 32) or cols > (1 << 32):
                raise MatrixFileError(f"implausible dimensions in {path}")
            vals = np.fromfile(f, dtype="<f8", count=rows * cols)
    except OSError as e:
        raise MatrixFileError(f"cannot open: {path}") from e
    if vals.size != rows * cols:
        raise MatrixFileError(f"truncated matrix file: {path}")
    fmt = FORMATS[fmt_id]
    return quantize_array(vals.reshape(rows, cols).astype(np.float64), fmt), fmt


def save_matrix_csv(values: np.ndarray, path: str) -> None:
    """save_matrix_csv (matrix_io.cpp:90-101): precision 17."""
    v = np.asarray(values, dtype=np.float64)
    try:
        with open(path, "w") as f:
            for row in v:
                f.write(",".join(format(float(x), ".17g") for x in row) + "\n")
    except OSError as e:
        raise MatrixFileError(f"cannot open for writing: {path}") from e


def load_matrix_csv(path: str, fmt: str) -> np.ndarray:
    """load_matrix_csv (matrix_io.cpp:103-125)."""
    rows, cols = [], -1
    try:
        with open(path) as f:
            for line in f:
                line = line.rstrip("\n")
                if not line:
                    continue
                toks = [t for t in line.split(",")]
                try:
                    vals = [float(t) for t in toks if t != ""]
                except ValueError as e:
                    raise _capi.InvalidArgument(f"bad CSV number in {path}") from e  # std::stod
                if cols == -1:
                    cols = len(vals)
                elif len(vals) != cols:
                    raise MatrixFileError(f"ragged CSV row in {path}")
                rows.append(vals)
    except OSError as e:
        raise MatrixFileError(f"cannot open: {path}") from e
    if not rows:
        raise MatrixFileError(f"empty CSV: {path}")
    return quantize_array(np.array(rows, dtype=np.float64), fmt)


def load_matrix_auto(path: str, csv_format: Optional[str] = None) -> Tuple[np.ndarray, str]:
    """load_matrix_auto (matrix_io.cpp:127-137)."""
    try:
        with open(path, "rb") as f:
            magic = f.read(8)
    except OSError as e:
        raise MatrixFileError(f"cannot open: {path}") from e
    if magic == MAGIC:
        return load_matrix_binary(path)
    fmt = csv_format or "fp64"
    return load_matrix_csv(path, fmt), fmt


def verify_files(a_path: str, b_path: str, check_against: Optional[str] = None, precision: str = "fp64",
                 mode: str = "offline", e_max: Optional[float] = None, c_sigma: float = 2.5,
                 engine: str = "exact"):
    """verify_files (harness.cpp:430-490) on the GPU. Returns (json dict,
    exit code). precision is the format CSV inputs are quantized into
    (ExperimentConfig::precision); e_max defaults to the format model at
    dim = K (resolve_e_max). engine="exact" reproduces the reference bit for
    bit; engine="tensor" runs the tcgen05 kernel (BF16/FP16, FP32
    NativeBlocked(128) checksums) for large real-weight files."""
    t0 = time.perf_counter()
    a, fa = load_matrix_auto(a_path, precision)
    b, fb = load_matrix_auto(b_path, precision)
    if a.shape[1] != b.shape[0]:
        raise _capi.InvalidArgument("verify: A's columns must equal B's rows")
    if fa != fb:
        raise _capi.InvalidArgument("verify: operand precisions disagree")
    prod = api.encode_and_multiply(a, b, mode, fa, engine=engine)
    if check_against is not None:
        c, fc = load_matrix_auto(check_against, fa)
        if c.shape != prod.c.shape:
            raise _capi.InvalidArgument("verify: --check-against dimensions disagree")
        if fc != fa:
            raise _capi.InvalidArgument("verify: --check-against precision disagrees")
        prod.c = c
        prod.c_accum = c  # verified as stored (on-grid values: exact in the FP32 source storage)
    k = a.shape[1]
    e = e_max if e_max is not None else api.resolve_e_max(fa, k)
    T = api.vabft_thresholds(a, b, api.VabftParams(e, c_sigma), fa)
    verdicts = api.verify(prod, T)
    rows = []
    for v in verdicts:
        if not v.detected:
            continue
        r = {"row": v.row, "diff1": v.diff1 if math.isfinite(v.diff1) else None, "threshold": v.threshold}
        if v.location is not None:
            r.update({"location": v.location, "residual": v.localization_residual, "correction": v.correction})
        rows.append(r)
    doc = {"a": a_path, "b": b_path, "dims": [a.shape[0], a.shape[1], b.shape[1]], "precision": fa, "mode": mode,
           "e_max": {"value": e, "source": "override" if e_max is not None else "format-default"},
           "c_sigma": c_sigma, "engine": engine}
    if check_against is not None:
        doc["check_against"] = check_against
    doc["detected"] = bool(rows)
    doc["detected_rows"] = rows
    doc["wall_time_s"] = time.perf_counter() - t0
    return doc, (2 if rows else 0)


def main(argv=None) -> int:
    """`python -m paper_2602_08043_b200.matrix_io verify A B [--check-against C] ...`"""
    import argparse
    import json
    ap = argparse.ArgumentParser(description="verify_files on the B200 path")
    ap.add_argument("a")
    ap.add_argument("b")
    ap.add_argument("--check-against")
    ap.add_argument("--precision", default="fp64", choices=FORMATS)
    ap.add_argument("--mode", default="offline", choices=["offline", "online"])
    ap.add_argument("--e-max", type=float)
    ap.add_argument("--c-sigma", type=float, default=2.5)
    ap.add_argument("--engine", default="exact", choices=["exact", "tensor"])
    args = ap.parse_args(argv)
    doc, code = verify_files(args.a, args.b, args.check_against, args.precision, args.mode, args.e_max,
                             args.c_sigma, args.engine)
    print(json.dumps(doc, indent=2))
    return code


if __name__ == "__main__":
    raise SystemExit(main())
