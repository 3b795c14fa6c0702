"""GPU parity of the CUDA path (through the C-ABI) against the reference's
golden vectors and the oracle.

Bars (BASELINE north star):
  EXACT engine  — C, C_accum, checksums, row sums, verdicts: bit-exact.
  stats/thresholds — within 1e-12 relative (bit-exact fraction reported).
  TENSOR engine — C_accum within the FP32-accumulate bound of
                  test_precision.cpp:181-206; checksums/row sums/verdicts
                  bit-exact against the oracle given the device accumulator.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FMTS = ["bf16", "fp16", "fp32", "fp64"]
SHAPES = [(8, 12, 10), (33, 70, 129), (64, 128, 96)]


def bits(x):
    return np.asarray(x, dtype=np.float64).view(np.uint64)


def same(a, b):
    """Bit-identical, except that any NaN equals any NaN (the x86 default NaN
    and the GPU canonical NaN differ only in sign/payload bits)."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and np.array_equal(bits(a[~na]), bits(b[~nb]))


@pytest.fixture(scope="module")
def api():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2602_08043_b200 import api as _api
    return _api


# ------------------------------------------------------------ EXACT engine
@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("mode", ["offline", "online"])
@pytest.mark.parametrize("si", range(len(SHAPES)))
def test_exact_encode_and_multiply_bitexact(api, golden, fmt, mode, si):
    A, B = golden[f"A_{fmt}_{si}"], golden[f"B_{fmt}_{si}"]
    e = api.encode_and_multiply(A, B, mode, fmt, engine="exact")
    key = f"{fmt}_{mode}_{si}"
    assert same(e.c, golden[f"C_{key}"])
    assert same(e.c_accum, golden[f"Ca_{key}"])
    assert same(e.row_check1, golden[f"rc1_{key}"])
    assert same(e.row_check2, golden[f"rc2_{key}"])
    assert same(e.col_check1, golden[f"cc1_{key}"])
    assert same(e.col_check2, golden[f"cc2_{key}"])
    r1, r2 = api.row_sums(e.verification_source(), e.checksum_precision, e.verification_format())
    assert same(r1, golden[f"rs1_{key}"]) and same(r2, golden[f"rs2_{key}"])


@pytest.mark.parametrize("fmt", ["fp32", "fp64"])
@pytest.mark.parametrize("kind", [1, 2, 3])
def test_exact_strategies_match_oracle(api, port, fmt, kind):
    # every AccumKind for the native formats, including non-power-of-two K (H9)
    A, B = port.trial_inputs(19, 203, 37, fmt, "normal:0,1", 9, kind)
    spec = api.PrecisionSpec.of(fmt).with_accumulation(api.AccumStrategy(kind, 16))
    e = api.encode_and_multiply(A, B, "offline", spec, engine="exact")
    o = port.encode_and_multiply(A, B, fmt, "offline", accum=(kind, 16))
    assert same(e.c_accum, o.c_accum) and same(e.c, o.c)
    assert same(e.row_check1, o.row_check1) and same(e.row_check2, o.row_check2)
    assert same(e.col_check1, o.col_check1) and same(e.col_check2, o.col_check2)


def test_exact_larger_bf16_matches_oracle(api, port):
    A, B = port.trial_inputs(130, 1030, 260, "bf16", "normal:0,1", 4, 2)
    for mode in ("offline", "online"):
        e = api.encode_and_multiply(A, B, mode, "bf16", engine="exact")
        o = port.encode_and_multiply(A, B, "bf16", mode)
        assert same(e.c, o.c) and same(e.c_accum, o.c_accum)
        assert same(e.row_check1, o.row_check1) and same(e.row_check2, o.row_check2)


# --------------------------------------------------------------- stats
@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("si", range(len(SHAPES)))
def test_thresholds_match_reference(api, golden, fmt, si):
    A, B = golden[f"A_{fmt}_{si}"], golden[f"B_{fmt}_{si}"]
    e_max = float(golden[f"emax_{fmt}_{si}"][0])
    T, s = api.vabft_thresholds(A, B, api.VabftParams(e_max, 2.5), fmt, return_summary=True)
    ref_T = golden[f"T_{fmt}_{si}"]
    assert same(s, golden[f"bsum_{fmt}_{si}"])  # sequential k-order sums: bit-exact
    np.testing.assert_allclose(T, ref_T, rtol=1e-12, atol=0)
    at = api.aabft_threshold(A, B, api.AabftParams.for_format(fmt), fmt)
    np.testing.assert_allclose(at.per_row, golden[f"Ta_{fmt}_{si}"], rtol=1e-12, atol=0)


def test_row_stats_known(api):
    s = api.row_stats(np.full(1000, 3.5))
    assert s.mean == 3.5 and s.var_bound == 0.0
    s = api.row_stats([-1.0, 1.0])
    assert s.mean == 0.0 and s.var_bound == 1.0
    s = api.row_stats(np.full(10**6, 0.1))
    assert abs(s.mean - 0.1) < 1e-15
    with pytest.raises(ValueError):
        api.row_stats([1.0, math.inf])


def test_row_stats_bitexact_fraction(api, ref_or_port):
    rng = np.random.default_rng(3)
    X = rng.standard_normal((512, 777)).astype(np.float32).astype(np.float64)
    mean, mx, mn, vb = api._row_stats_matrix(X, "fp32")
    ref = np.array([ref_or_port.row_stats(r) for r in X])
    assert np.array_equal(mx, ref[:, 1]) and np.array_equal(mn, ref[:, 2])
    np.testing.assert_allclose(mean, ref[:, 0], rtol=1e-13, atol=1e-300)
    assert np.mean(mean == ref[:, 0]) >= 0.99


# -------------------------------------------------------------- verify
@pytest.mark.parametrize("mode", ["offline", "online"])
def test_verify_golden(api, golden, mode):
    cs = api.checksum_precision_for("fp32", mode)
    v = api.verify_arrays(golden[f"vsrc_{mode}"], "fp32", golden[f"vrc1_{mode}"], golden[f"vrc2_{mode}"],
                          golden[f"vT_{mode}"], cs)
    for k in ("diff1", "diff2", "residual"):
        assert same(v[k], golden[f"v{k}_{mode}"]), k
    assert np.array_equal(v["detected"], golden[f"vdetected_{mode}"].astype(bool))
    assert np.array_equal(v["location"], golden[f"vlocation_{mode}"])
    assert v["counts"][0] == 16 and v["counts"][1] == golden[f"vdetected_{mode}"].sum()


def test_verify_rejects_negative_thresholds(api, golden):
    cs = api.checksum_precision_for("fp32", "offline")
    with pytest.raises(ValueError):
        api.verify_arrays(golden["vsrc_offline"], "fp32", golden["vrc1_offline"], golden["vrc2_offline"],
                          -np.ones(16), cs)


def test_localize_matches(api, golden):
    for (d1, d2, n), (j, r) in zip(golden["loc_cases"], golden["loc_out"]):
        got = api.localize(d1, d2, int(n))
        assert (got is None) if j < 0 else (got == (int(j), r))


# -------------------------------------------------------------- inject
@pytest.mark.parametrize("fmt", FMTS)
def test_inject_fixed_positions(api, golden, fmt):
    A = golden[f"inj_in_{fmt}"]
    for rep, rec in enumerate(golden[f"inj_rec_{fmt}"]):
        i, j, applied, dtaken, bit, d, pos_mode = (int(x) for x in rec)
        if i < 0:
            continue
        X, r = api.inject(A, fmt, api.FaultSpec((i, j), bit, dtaken))
        assert same(X, golden[f"inj_out_{fmt}"][rep]) and r.applied == bool(applied)


# -------------------------------------------------------------- TENSOR engine
@pytest.mark.parametrize("fmt", ["bf16", "fp16"])
@pytest.mark.parametrize("mode", ["offline", "online"])
@pytest.mark.parametrize("shape", [(64, 128, 96), (200, 264, 72), (256, 512, 384)])
def test_tensor_engine_parity(api, port, fmt, mode, shape):
    m, k, n = shape
    A, B = port.trial_inputs(m, k, n, fmt, "normal:0,1", 11, 1)
    e = api.encode_and_multiply(A, B, mode, fmt, engine="tensor")
    o = port.encode_and_multiply(A, B, fmt, mode)
    # C_accum within the FP32 accumulation bound (test_precision.cpp:181-206)
    bound = (k + 1) * 2.0**-24 * (np.abs(A) @ np.abs(B))
    assert np.all(np.abs(e.c_accum - o.c_accum) <= bound)
    # C is the quantized accumulator (RNE, saturating)
    q = np.array([port.quantize(x, fmt) for x in e.c_accum.ravel()]).reshape(e.c.shape)
    assert same(e.c, q)
    # checksums: FP32 blocked:128 order, bit-exact against the restatement
    blk = _blocked_checksums(port, A, B, fmt, mode)
    assert same(e.row_check1, blk[0]) and same(e.row_check2, blk[1])
    # row sums of the device accumulator / output == reference row_sums with
    # an FP32 NativeBlocked(128) sum precision
    src = e.verification_source()
    r1, r2 = api.row_sums(src, e.checksum_precision, e.verification_format())
    p1, p2 = port.row_sums(src, "fp32", "offline", accum=(2, 128))
    assert same(r1, p1) and same(r2, p2)
    # verdicts on planted faults: device verify == oracle verify (same inputs)
    src2 = src.copy()
    src2[1, 3] += 7.0
    src2[5, n - 1] = -src2[5, n - 1] * 9.0 + 1.0
    T = np.full(m, 1e-3)
    v = api.verify_arrays(src2, "fp32", e.row_check1, e.row_check2, T, e.checksum_precision)
    o = port.verify(src2, e.row_check1, e.row_check2, T, "fp32", "offline", accum=(2, 128))
    assert same(v["diff1"], o["diff1"]) and same(v["diff2"], o["diff2"])
    assert np.array_equal(v["detected"], o["detected"]) and np.array_equal(v["location"], o["location"])


def _blocked_checksums(port, A, B, fmt, mode):
    """Row checksums A (B r) with the blocked:128 strategy, restated from
    encode_impl (checksum.cpp:103-146) with float working type."""
    f32 = np.float32
    Bf = B.astype(f32)
    n = B.shape[1]
    w = np.arange(1, n + 1, dtype=f32)

    def blocked(terms):
        tot = f32(0)
        for b0 in range(0, terms.shape[-1], 128):
            part = f32(0)
            for t in terms[b0:b0 + 128]:
                part = f32(part + t)
            tot = f32(tot + part)
        return tot

    br1 = np.array([blocked(Bf[q]) for q in range(B.shape[0])], dtype=f32)
    br2 = np.array([blocked((w * Bf[q]).astype(f32)) for q in range(B.shape[0])], dtype=f32)
    if mode == "offline":
        br1 = np.array([port.quantize(float(x), fmt) for x in br1], dtype=f32)
        br2 = np.array([port.quantize(float(x), fmt) for x in br2], dtype=f32)
    Af = A.astype(f32)
    c1 = np.array([blocked((br1 * Af[i]).astype(f32)) for i in range(A.shape[0])], dtype=np.float64)
    c2 = np.array([blocked((br2 * Af[i]).astype(f32)) for i in range(A.shape[0])], dtype=np.float64)
    if mode == "offline":
        c1 = np.array([port.quantize(x, fmt) for x in c1])
        c2 = np.array([port.quantize(x, fmt) for x in c2])
    return c1, c2


def test_plain_gemm_matches_torch(api):
    import torch
    from paper_2602_08043_b200 import _capi
    from paper_2602_08043_b200.device import ptr, stream_ptr
    torch.manual_seed(0)
    for (m, n, k) in [(128, 256, 64), (200, 264, 72), (1024, 768, 768)]:
        for kmaj in (0, 1):
            a = torch.randn(m, k, device="cuda").bfloat16()
            b = torch.randn(k, n, device="cuda").bfloat16()
            bb = b.t().contiguous() if kmaj else b
            c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
            _capi.check(_capi.lib.vabft_gemm_plain(0, kmaj, m, n, k, ptr(a), ptr(bb), ptr(c), stream_ptr()))
            ref = a.float() @ b.float()
            bound = (k + 1) * 2.0**-24 * (a.float().abs() @ b.float().abs()) + ref.abs() * 2.0**-8
            assert bool(((c.float() - ref).abs() <= bound).all())


def test_plain_gemm_pair_split_last_wave_matches_one_cta(api):
    """Plain GEMM at shapes whose last pair wave runs as 128-column half tiles
    (4096 x 4096: 256 pair tiles over 74 pairs; 2560 x 4000 ragged): C is
    bit-identical to the one-CTA kernel's."""
    import torch
    from paper_2602_08043_b200 import _capi
    from paper_2602_08043_b200.device import ptr, stream_ptr
    torch.manual_seed(1)
    for (m, n, k) in [(4096, 4096, 256), (2560, 4000, 128)]:
        a = torch.randn(m, k, device="cuda").bfloat16()
        b = torch.randn(k, n, device="cuda").bfloat16()
        out = []
        for mode in (0, 1):
            c = torch.full((m, n), float("nan"), device="cuda", dtype=torch.bfloat16)
            _capi.check(_capi.lib.vabft_gemm_plain_mode(0, 0, m, n, k, ptr(a), ptr(b), ptr(c), mode, stream_ptr()))
            out.append(c)
        torch.cuda.synchronize()
        assert torch.equal(out[0].view(torch.int16), out[1].view(torch.int16))


def test_aabft_fixed_y_zero_and_negative_keep_reference_semantics(api):
    """AabftParams::fixed_y = 0 (or negative) is a fixed y in the reference
    (threshold_aabft.cpp:50-60): y_used = that value, degenerate = (y == 0),
    thresholds = confidence * sigma(K, t, y); only an empty fixed_y computes y
    (the C-ABI's NaN sentinel)."""
    A = np.ones((4, 8))
    B = np.ones((8, 5))
    z = api.aabft_threshold(A, B, api.AabftParams(23, 0.0, 3.0), "fp32")
    assert z.y_used == 0.0 and z.degenerate and np.all(z.per_row == 0.0)
    neg = api.aabft_threshold(A, B, api.AabftParams(23, -2.0, 3.0), "fp32")
    assert neg.y_used == -2.0 and not neg.degenerate and np.all(neg.per_row < 0.0)
    assert neg.per_row[0] == 3.0 * api.aabft_sigma(8, 23, -2.0)
    comp = api.aabft_threshold(A, B, api.AabftParams(23, None, 3.0), "fp32")
    assert comp.y_used == 1.0 * 5.0  # max|A| * max_k |sum_j B[k][j]|
