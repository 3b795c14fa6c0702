"""TEST INFRASTRUCTURE ONLY — CPU oracles for the V-ABFT hot path.

Two interchangeable backends with identical Python signatures:

* ``port()``  — oracle/build/libvabft_oracle.so, the plain-C restatement
  (oracle/vabft_oracle.c) of the reference algorithm, every function citing
  the reference file:line it follows.
* ``ref()``   — oracle/_ref/libvabft_ref.so, the UNMODIFIED reference C++
  sources compiled by oracle/Makefile plus the extern "C" adapter
  oracle/ref_shim.cpp (available wherever that .so was built; it travels to
  the GPU box with the repo snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
reference arm may import this package, and only as the checker. The product
package ``paper_2602_08043_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "build", "libvabft_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libvabft_ref.so")

FORMATS = {"bf16": 0, "fp16": 1, "fp32": 2, "fp64": 3}
DISTS = {"normal": 0, "uniform": 1, "truncnormal": 2, "absnormal": 3}

_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_U64 = C.POINTER(C.c_uint64)
_U32 = C.POINTER(C.c_uint32)
_U8 = C.POINTER(C.c_uint8)
i64 = C.c_int64
u64 = C.c_uint64
dbl = C.c_double
cint = C.c_int


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _dp(a):
    return None if a is None else a.ctypes.data_as(_D)


def _arr(x, dtype=np.float64):
    return np.ascontiguousarray(x, dtype=dtype)


def parse_dist(text: str):
    """Distribution::parse (proj/src/distribution.cpp:75-93)."""
    name, _, rest = text.partition(":")
    args = [float(t) for t in rest.split(",") if t] if rest else []
    arg = lambda i, d: args[i] if i < len(args) else d  # noqa: E731
    if name == "normal":
        return (0, arg(0, 0.0), arg(1, 1.0), -1.0, 1.0)
    if name == "uniform":
        return (1, arg(0, -1.0), arg(1, 1.0), -1.0, 1.0)
    if name == "truncnormal":
        return (2, arg(0, 0.0), arg(1, 1.0), arg(2, -1.0), arg(3, 1.0))
    if name == "absnormal":
        return (3, arg(0, 1.0), arg(1, 1.0), -1.0, 1.0)
    raise ValueError(f"unknown distribution: {text}")


@dataclass
class Encoded:
    c: np.ndarray
    c_accum: np.ndarray
    row_check1: np.ndarray
    row_check2: np.ndarray
    col_check1: np.ndarray
    col_check2: np.ndarray


class Oracle:
    """ctypes binding of one backend; `p` is the symbol prefix."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library not built: {path} (run make -C oracle)")
        self.path = path
        self.lib = C.CDLL(path)
        self.p = prefix
        self.name = "reference" if prefix == "ref_" else "port"
        L = self.lib
        f = lambda n: getattr(L, prefix + n)  # noqa: E731
        self._err = f("last_error")
        self._err.restype = C.c_char_p
        sig = {
            "philox_block": (None, [_U32, _U32, _U32]),
            "philox_draws": (cint, [u64, u64, cint, dbl, i64, _D, _U64]),
            "trial_inputs": (cint, [i64, i64, i64, cint, cint, dbl, dbl, dbl, dbl, u64, u64, _D, _D]),
            "quantize": (cint, [dbl, cint, cint, _D]),
            "encode_and_multiply": (cint, [cint, cint, i64, cint, i64, i64, i64, _D, _D, _D, _D, _D, _D, _D, _D]),
            "row_sums": (cint, [cint, cint, cint, i64, i64, i64, _D, _D, _D]),
            "row_stats": (cint, [_D, i64, _D]),
            "threshold_row": None,
            "vabft_thresholds": (cint, [cint, i64, i64, i64, _D, _D, dbl, dbl, _D, _D]),
            "resolve_e_max": (cint, [cint, i64, _D]),
            "aabft_sigma": (cint, [i64, cint, dbl, _D]),
            "aabft_threshold": (cint, [cint, i64, i64, i64, _D, _D, cint, dbl, dbl, _D, _D, C.POINTER(cint)]),
            "localize": (cint, [dbl, dbl, i64, _I64, _D]),
            "verify": (cint, [cint, cint, cint, i64, i64, i64, _D, _D, _D, _D, dbl, _D, _D, _U8, _I64, _D]),
            "encode_bits": (cint, [dbl, cint, _U64]),
            "decode_bits": (cint, [u64, cint, _D]),
            "inject": (cint, [cint, cint, i64, i64, _D, i64, i64, cint, cint, u64, u64, _I64, _D]),
            "campaign_trial": (cint, [i64, i64, i64, cint, cint, dbl, dbl, dbl, dbl, cint, cint, u64, u64, cint, cint, dbl, dbl, _I64]),
        }
        for name, s in sig.items():
            if s is None:
                continue
            fn = f(name)
            fn.restype, fn.argtypes = s
        if prefix == "ref_":
            L.ref_threshold_row.restype = cint
            L.ref_threshold_row.argtypes = [_D, _D, i64, i64, dbl, dbl, _D]
            L.ref_injection_campaign.restype = cint
            L.ref_injection_campaign.argtypes = [i64, i64, i64, cint, cint, dbl, dbl, dbl, dbl, cint, cint, i64, u64, cint, cint, dbl, dbl, _I64]
            L.ref_calibrate.restype = cint
            L.ref_calibrate.argtypes = [cint, cint, _I64, i64, i64, u64, i64, _D, _D]
            L.ref_correct.restype = cint
            L.ref_correct.argtypes = [cint, i64, i64, _D, i64, i64, dbl, _D]
            L.ref_max_threads.restype = cint
            L.ref_save_matrix.restype = cint
            L.ref_save_matrix.argtypes = [cint, cint, i64, i64, _D, C.c_char_p]
            L.ref_load_matrix.restype = cint
            L.ref_load_matrix.argtypes = [C.c_char_p, cint, _I64, _D]
        else:
            L.vo_threshold_row.restype = cint
            L.vo_threshold_row.argtypes = [_D, _D, i64, dbl, dbl, _D]

    def _call(self, name, *args):
        rc = getattr(self.lib, self.p + name)(*args)
        if rc:
            raise OracleError(rc, self._err().decode())

    # ---------------------------------------------------------------- rng
    def philox_block(self, ctr, key):
        c = (C.c_uint32 * 4)(*ctr)
        k = (C.c_uint32 * 2)(*key)
        o = (C.c_uint32 * 4)()
        getattr(self.lib, self.p + "philox_block")(c, k, o)
        return list(o)

    def draws(self, seed, stream, kind, count, arg=0.0):
        out = np.zeros(count)
        outu = np.zeros(count, dtype=np.uint64)
        self._call("philox_draws", seed, stream, kind, arg, count, _dp(out), outu.ctypes.data_as(_U64))
        return outu if kind in (0, 1, 4) else out

    def trial_inputs(self, m, k, n, fmt, dist, seed, stream, with_b=True):
        kind, p0, p1, lo, hi = parse_dist(dist) if isinstance(dist, str) else dist
        A = np.zeros((m, k))
        B = np.zeros((k, n)) if with_b else None
        self._call("trial_inputs", m, k, n, FORMATS[fmt], kind, p0, p1, lo, hi, seed, stream, _dp(A), _dp(B))
        return A, B

    # ---------------------------------------------------------- precision
    def quantize(self, x, fmt, overflow_error=False):
        out = C.c_double()
        self._call("quantize", float(x), FORMATS[fmt], int(overflow_error), C.byref(out))
        return out.value

    def encode_and_multiply(self, A, B, fmt, mode="offline", accum=None):
        A = _arr(A)
        B = _arr(B)
        m, k = A.shape
        n = B.shape[1]
        kind, bl = (-1, 128) if accum is None else accum
        c = np.zeros((m, n))
        ca = np.zeros((m, n))
        r1, r2 = np.zeros(m), np.zeros(m)
        c1, c2 = np.zeros(n), np.zeros(n)
        self._call("encode_and_multiply", FORMATS[fmt], kind, bl, 1 if mode == "online" else 0, m, k, n,
                   _dp(A), _dp(B), _dp(c), _dp(ca), _dp(r1), _dp(r2), _dp(c1), _dp(c2))
        return Encoded(c, ca, r1, r2, c1, c2)

    def row_sums(self, src, fmt, mode="offline", accum=None):
        src = _arr(src)
        m, n = src.shape
        kind, bl = (-1, 128) if accum is None else accum
        r1, r2 = np.zeros(m), np.zeros(m)
        self._call("row_sums", FORMATS[fmt], 1 if mode == "online" else 0, kind, bl, m, n, _dp(src), _dp(r1), _dp(r2))
        return r1, r2

    def blocked_row_checksums(self, A, B, fmt, mode="online", block=128):
        """Row checksums A (B r1), A (B r2) of encode_impl (checksum.cpp:103-115,
        129-134) in the fused path's checksum precision — the accumulator's
        working type (FP32 for BF16/FP16/FP32, FP64 for FP64) in
        NativeBlocked(block) order — composed from this backend's own row_sums
        (checksum.cpp:160-187) without the emulated GEMM:
          B r1, B r2      = row_sums(B)                       (over j, weights j+1)
          offline         : quantize both to the input format (checksum.cpp:112-115)
          A (B r)[i]      = row_sums(P)[i], P[i][k] = fl_T(br[k] * A[i][k])
                            (the contract's products, rounded in T, checksum.cpp:74-79)
          offline         : quantize to the input format (checksum.cpp:129-134)."""
        wt = np.float64 if fmt == "fp64" else np.float32
        wf = "fp64" if fmt == "fp64" else "fp32"
        br1, br2 = self.row_sums(B, wf, "offline", accum=(2, block))
        if mode == "offline":
            br1 = np.array([self.quantize(x, fmt) for x in br1])
            br2 = np.array([self.quantize(x, fmt) for x in br2])
        Aw = _arr(A).astype(wt)
        out = []
        for br in (br1, br2):
            P = (br.astype(wt)[None, :] * Aw).astype(np.float64)
            c, _ = self.row_sums(P, wf, "offline", accum=(2, block))
            if mode == "offline":
                c = np.array([self.quantize(x, fmt) for x in c])
            out.append(c)
        return out[0], out[1]

    def row_stats(self, v):
        v = _arr(v)
        out = np.zeros(5)
        self._call("row_stats", _dp(v), v.size, _dp(out))
        return out

    def threshold_row(self, a_stats, b_summary, n, e_max, c_sigma=2.5, k_len=1):
        a = _arr(a_stats)
        b = _arr(b_summary)
        out = np.zeros(4)
        if self.p == "ref_":
            self._call("threshold_row", _dp(a), _dp(b), k_len, n, e_max, c_sigma, _dp(out))
        else:
            self._call("threshold_row", _dp(a), _dp(b), n, e_max, c_sigma, _dp(out))
        return out

    def vabft_thresholds(self, A, B, e_max, c_sigma=2.5, fmt="fp64"):
        A, B = _arr(A), _arr(B)
        m, k = A.shape
        n = B.shape[1]
        T = np.zeros(m)
        s = np.zeros(3)
        self._call("vabft_thresholds", FORMATS[fmt], m, k, n, _dp(A), _dp(B), e_max, c_sigma, _dp(T), _dp(s))
        return T, s

    def resolve_e_max(self, fmt, dim):
        out = C.c_double()
        self._call("resolve_e_max", FORMATS[fmt], dim, C.byref(out))
        return out.value

    def aabft_sigma(self, n, t, y):
        out = C.c_double()
        self._call("aabft_sigma", n, t, y, C.byref(out))
        return out.value

    def aabft_threshold(self, A, B, fmt, mantissa_bits=-1, fixed_y=None, conf=3.0, computed=None):
        """fixed_y=None means the format default (21 for FP32/FP64, computed for 16-bit)."""
        A, B = _arr(A), _arr(B)
        m, k = A.shape
        n = B.shape[1]
        if fixed_y is None:
            fixed_y = 21.0 if fmt in ("fp32", "fp64") else math.nan
        if computed:
            fixed_y = math.nan
        T = np.zeros(m)
        y = C.c_double()
        dg = C.c_int()
        self._call("aabft_threshold", FORMATS[fmt], m, k, n, _dp(A), _dp(B), mantissa_bits, fixed_y, conf,
                   _dp(T), C.byref(y), C.byref(dg))
        return T, y.value, bool(dg.value)

    # -------------------------------------------------------------- detect
    def localize(self, d1, d2, n_cols):
        j = C.c_int64()
        r = C.c_double()
        ok = getattr(self.lib, self.p + "localize")(d1, d2, n_cols, C.byref(j), C.byref(r))
        return (j.value, r.value) if ok else None

    def verify(self, source, rc1, rc2, T, fmt, mode="offline", accum=None, floor_scale=1e-3):
        source = _arr(source)
        m, n = source.shape
        kind, bl = (-1, 128) if accum is None else accum
        rc1, rc2, T = _arr(rc1), _arr(rc2), _arr(T)
        d1, d2, res = np.zeros(m), np.zeros(m), np.zeros(m)
        det = np.zeros(m, dtype=np.uint8)
        loc = np.zeros(m, dtype=np.int64)
        self._call("verify", FORMATS[fmt], 1 if mode == "online" else 0, kind, bl, m, n, _dp(source), _dp(rc1),
                   _dp(rc2), _dp(T), floor_scale, _dp(d1), _dp(d2), det.ctypes.data_as(_U8),
                   loc.ctypes.data_as(_I64), _dp(res))
        return {"diff1": d1, "diff2": d2, "detected": det.astype(bool), "location": loc, "residual": res}

    # -------------------------------------------------------------- faults
    def encode_bits(self, v, fmt):
        out = C.c_uint64()
        self._call("encode_bits", float(v), FORMATS[fmt], C.byref(out))
        return out.value

    def decode_bits(self, b, fmt):
        out = C.c_double()
        self._call("decode_bits", int(b), FORMATS[fmt], C.byref(out))
        return out.value

    def inject(self, X, fmt, bit, direction=0, pos=None, seed=0, stream=0, src_fp32=False):
        X = _arr(X).copy()
        m, n = X.shape
        rec = np.zeros(4, dtype=np.int64)
        vals = np.zeros(2)
        pi, pj = pos if pos is not None else (-1, -1)
        self._call("inject", FORMATS[fmt], int(src_fp32), m, n, _dp(X), pi, pj, bit, direction, seed, stream,
                   rec.ctypes.data_as(_I64), _dp(vals))
        return X, {"i": int(rec[0]), "j": int(rec[1]), "applied": bool(rec[2]), "direction_taken": int(rec[3]),
                   "value_before": vals[0], "value_after": vals[1]}

    def calibrate(self, fmt, sizes, trials, seed, mode="offline", dim=None):
        """Reference calibrate (calibration.cpp:88-150); reference library only.
        Returns (maxima, {kind, value, scale, offset, recommended, e_max_at_dim})."""
        if self.name != "reference":
            raise OracleError(5, "calibrate: reference library only")
        sz = np.asarray(sizes, dtype=np.int64)
        mx = np.zeros(len(sizes))
        out = np.zeros(6)
        self._call("calibrate", FORMATS[fmt], 1 if mode == "online" else 0, sz.ctypes.data_as(_I64), len(sizes), trials, seed,
                   int(dim if dim is not None else sizes[-1]), _dp(mx), _dp(out))
        return mx, {"kind": "constant" if out[0] == 0.0 else "sqrt_scaled", "value": out[1], "scale": out[2],
                    "offset": out[3], "recommended": out[4], "e_max_at_dim": out[5]}

    def injection_campaign(self, m, k, n, fmt, dist, bit, trials, seed, mode="offline", method=0, e_max=8e-3,
                           c_sigma=2.5, direction=1):
        """Reference injection_campaign (faults.cpp:170-216), multithreaded over
        trials; reference library only. Returns [trials, applicable, detected,
        located_correctly, nonfinite_after]."""
        if self.name != "reference":
            raise OracleError(5, "injection_campaign: reference library only")
        kind, p0, p1, lo, hi = parse_dist(dist)
        out = np.zeros(5, dtype=np.int64)
        self._call("injection_campaign", m, k, n, FORMATS[fmt], kind, p0, p1, lo, hi, bit, direction, trials, seed,
                   1 if mode == "online" else 0, method, e_max, c_sigma, out.ctypes.data_as(_I64))
        return out

    def save_matrix(self, X, fmt, path, binary=True):
        """Reference save_matrix_binary / save_matrix_csv (matrix_io.cpp:49-101); reference only."""
        X = _arr(X)
        self._call("save_matrix", int(binary), FORMATS[fmt], X.shape[0], X.shape[1], _dp(X), path.encode())

    def load_matrix(self, path, csv_fmt="fp64"):
        """Reference load_matrix_auto (matrix_io.cpp:127-137) -> (values, format); reference only."""
        dims = np.zeros(3, dtype=np.int64)
        self._call("load_matrix", path.encode(), FORMATS[csv_fmt], dims.ctypes.data_as(_I64), None)
        out = np.zeros((int(dims[0]), int(dims[1])))
        self._call("load_matrix", path.encode(), FORMATS[csv_fmt], dims.ctypes.data_as(_I64), _dp(out))
        return out, list(FORMATS)[int(dims[2])]

    def campaign_trial(self, m, k, n, fmt, dist, bit, seed, trial, mode="offline", method=0, e_max=8e-3,
                       c_sigma=2.5, direction=1):
        kind, p0, p1, lo, hi = parse_dist(dist)
        out = np.zeros(6, dtype=np.int64)
        self._call("campaign_trial", m, k, n, FORMATS[fmt], kind, p0, p1, lo, hi, bit, direction, seed, trial,
                   1 if mode == "online" else 0, method, e_max, c_sigma, out.ctypes.data_as(_I64))
        return out


_cache = {}


def port() -> Oracle:
    if "port" not in _cache:
        _cache["port"] = Oracle(PORT_SO, "vo_")
    return _cache["port"]


def ref() -> Oracle:
    if "ref" not in _cache:
        _cache["ref"] = Oracle(REF_SO, "ref_")
    return _cache["ref"]


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def best() -> Oracle:
    """The unmodified reference when built, else the restatement."""
    return ref() if have_ref() else port()
