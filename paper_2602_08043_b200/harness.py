"""Experiment runners around the hot path: the reference's
tightness and false-positive experiments (harness.cpp:175-351), run on the
device engines, with trial operands drawn from the reference's own Philox
streams (trial t uses Philox(seed, t): A then B, random_matrix) so a trial
here is the same trial as in the reference.

  run_tightness  mean threshold / mean actual |checksum - baseline row sum|
                 per method, rows not covered (actual > threshold)
  run_fpr        rows with isnan(D1) or |D1| > T on clean data

Actual differences (baseline_row_diffs, harness.cpp:50-63): FP64 sources use
the exactly rounded |row_check1 - sum_j c_ij| (math.fsum over the row and the
checksum: one rounding of the exact value, what the MPFR oracle computes);
other sources the reference's FP64 Kahan-Babuska compensated sum.

Methods: "vabft", "vabft-blockwise" (blockwise.py, tiles (tile_k, tile_n)),
"aabft-fixed-y", "aabft-computed-y". e_max: the override, else the format's
model at dim = K ("format-default"); the reference's default is a CPU
calibration (resolve_run_e_max), which the EXACT engine reproduces but is
not rerun here.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import api, blockwise

METHODS = ("vabft", "vabft-blockwise", "aabft-fixed-y", "aabft-computed-y")


@dataclass
class ExperimentConfig:
    """ExperimentConfig (harness.hpp:25-42), the fields the runners use."""
    precision: str = "fp32"
    dist: str = "uniform:-1,1"
    m: int = 128
    k: int = 1024
    n: int = 256
    trials: int = 100
    seed: int = 0
    methods: List[str] = field(default_factory=lambda: ["vabft"])
    mode: str = "offline"
    e_max_override: Optional[float] = None
    c_sigma: float = 2.5
    engine: str = "exact"
    tile_k: int = 1024
    tile_n: int = 256

    def echo(self, experiment: str) -> dict:
        return {"experiment": experiment, "precision": self.precision, "distribution": self.dist,
                "dims": [self.m, self.k, self.n], "trials": self.trials, "seed": self.seed, "mode": self.mode,
                "c_sigma": self.c_sigma, "rng": "philox4x32-10", "methods": list(self.methods),
                "engine": self.engine}


_SPEC = None


def trial_operands(cfg: ExperimentConfig, trial: int):
    """Philox(seed, trial) -> A (m x k) then B (k x n), random_matrix
    (distribution.cpp:95-101), via the C++ drop-in's generator."""
    from . import _core
    spec = {"bf16": _core.PrecisionSpec.bf16, "fp16": _core.PrecisionSpec.fp16, "fp32": _core.PrecisionSpec.fp32,
            "fp64": _core.PrecisionSpec.fp64}[cfg.precision]()
    rng = _core.Philox(cfg.seed, trial)
    d = _core.Distribution.parse(cfg.dist)
    a = _core.random_matrix(cfg.m, cfg.k, d, spec, rng).values()
    b = _core.random_matrix(cfg.k, cfg.n, d, spec, rng).values()
    return a, b


def compensated_sum_rows(x: np.ndarray) -> np.ndarray:
    """compensated_sum (harness.cpp:39-49) of every row, in column order."""
    s = np.zeros(x.shape[0])
    comp = np.zeros(x.shape[0])
    for j in range(x.shape[1]):
        v = x[:, j]
        t = s + v
        big = np.abs(s) >= np.abs(v)
        comp += np.where(big, (s - t) + v, (v - t) + s)
        s = t
    return s + comp


def baseline_row_diffs(prod: api.EncodedProduct) -> np.ndarray:
    """baseline_row_diffs (harness.cpp:50-63)."""
    src = prod.verification_source()
    if prod.verification_format() == "fp64":
        return np.array([abs(math.fsum([prod.row_check1[i]] + [-x for x in src[i]])) for i in range(src.shape[0])])
    return np.abs(prod.row_check1 - compensated_sum_rows(src))


def seq_mean(v) -> float:
    """sum / size with the reference's sequential FP64 loop (harness.cpp:205-208)."""
    s = 0.0
    for x in np.asarray(v, dtype=np.float64).tolist():
        s += x
    return s / len(v)


def resolve_e_max(cfg: ExperimentConfig) -> dict:
    if cfg.e_max_override is not None:
        return {"value": cfg.e_max_override, "source": "override"}
    return {"value": api.resolve_e_max(cfg.precision, cfg.k), "source": "format-default"}


def thresholds(cfg: ExperimentConfig, method: str, a: np.ndarray, b: np.ndarray, e_max: float) -> np.ndarray:
    """make_threshold_fn (harness.cpp:148-173) plus the block-wise method
    (per row: the largest block threshold, the bound of the row's worst block)."""
    if method == "vabft":
        return api.vabft_thresholds(a, b, api.VabftParams(e_max, cfg.c_sigma), cfg.precision)
    if method == "vabft-blockwise":
        e = cfg.e_max_override  # None: per-k-tile format model
        return blockwise.blockwise_thresholds(a, b, cfg.precision, cfg.tile_k, cfg.tile_n, e, cfg.c_sigma).max(axis=1)
    p = api.AabftParams.for_format(cfg.precision)
    if method == "aabft-fixed-y":
        p.fixed_y = 21.0
    elif method == "aabft-computed-y":
        p.fixed_y = None
    else:
        raise api._capi.InvalidArgument(f"unknown threshold method: {method}")
    return api.aabft_threshold(a, b, p, cfg.precision).per_row


def _encode(cfg, a, b):
    return api.encode_and_multiply(a, b, cfg.mode, cfg.precision, engine=cfg.engine)


def run_tightness(cfg: ExperimentConfig) -> dict:
    """run_tightness (harness.cpp:175-280)."""
    t0 = time.perf_counter()
    if cfg.precision == "fp64" and max(cfg.m, cfg.k, cfg.n) > 512:
        raise api._capi.InvalidArgument("FP64 tightness uses the high-precision oracle; cap dims at 512")
    em = resolve_e_max(cfg)
    mean_actual, max_actual = [], 0.0
    mthr: Dict[str, List[float]] = {mth: [] for mth in cfg.methods}
    uncovered = {mth: 0 for mth in cfg.methods}
    for trial in range(cfg.trials):
        a, b = trial_operands(cfg, trial)
        prod = _encode(cfg, a, b)
        actual = baseline_row_diffs(prod)
        mean_actual.append(seq_mean(actual))
        max_actual = max(max_actual, float(np.max(actual)))
        for mth in cfg.methods:
            thr = thresholds(cfg, mth, a, b, em["value"])
            mthr[mth].append(seq_mean(thr))
            uncovered[mth] += int(np.sum(actual > thr))
    ma = seq_mean(mean_actual)
    doc = {"config": cfg.echo("tightness"), "actual": {"mean": ma, "max": max_actual, "per_trial_mean": mean_actual}}
    doc["config"]["e_max"] = em
    doc["degenerate"] = ma == 0.0
    doc["methods"] = {}
    for mth in cfg.methods:
        mt = seq_mean(mthr[mth])
        doc["methods"][mth] = {"mean_threshold": mt, "per_trial_mean_threshold": mthr[mth],
                               "rows_not_covered": uncovered[mth], "tightness": None if ma == 0.0 else mt / ma}
    doc["wall_time_s"] = time.perf_counter() - t0
    return doc


def run_fpr(cfg: ExperimentConfig) -> dict:
    """run_fpr (harness.cpp:297-351)."""
    t0 = time.perf_counter()
    em = resolve_e_max(cfg)
    fp = {mth: [] for mth in cfg.methods}
    mthr = {mth: [] for mth in cfg.methods}
    max_d1 = 0.0
    for trial in range(cfg.trials):
        a, b = trial_operands(cfg, trial)
        prod = _encode(cfg, a, b)
        r1, _ = api.row_sums(prod.verification_source(), prod.checksum_precision, prod.verification_format())
        d1 = r1 - prod.row_check1
        max_d1 = max(max_d1, float(np.max(np.abs(d1))))
        for mth in cfg.methods:
            thr = thresholds(cfg, mth, a, b, em["value"])
            fp[mth].append(int(np.sum(np.isnan(d1) | (np.abs(d1) > thr))))
            mthr[mth].append(seq_mean(thr))
    doc = {"config": cfg.echo("fpr"), "max_abs_diff1": max_d1, "rows_per_trial": cfg.m, "methods": {}}
    doc["config"]["e_max"] = em
    for mth in cfg.methods:
        tot = sum(fp[mth])
        with_fp = sum(1 for x in fp[mth] if x > 0)
        doc["methods"][mth] = {"false_positive_rows": tot, "clean_rows": cfg.trials * cfg.m - tot,
                               "row_fpr": tot / (cfg.trials * cfg.m), "trials_with_false_positive": with_fp,
                               "trial_fpr": with_fp / cfg.trials, "mean_threshold": sum(mthr[mth]) / cfg.trials}
    doc["wall_time_s"] = time.perf_counter() - t0
    return doc
