"""The C++ drop-in (include/vabft_cpp.hpp) through its pybind11 module _core,
checked against the reference (oracle/_ref, else the port) the way the
reference's own unit tests check the library (proj/tests/unit/*).

CPU tests: host-side semantics (Philox / ziggurat streams, distributions,
quantize, bit codecs, localize, thresholds' scalar formulas, fault placement,
exception types) and that the device entry points refuse to run without a
GPU. GPU tests: every device-backed entry point bit-exact against the
reference on the same inputs, including a whole injection campaign."""
import math

import numpy as np
import pytest

core = pytest.importorskip("paper_2602_08043_b200._core")

FMTS = {"bf16": core.Format.BF16, "fp16": core.Format.FP16, "fp32": core.Format.FP32, "fp64": core.Format.FP64}
SPEC = {"bf16": core.PrecisionSpec.bf16, "fp16": core.PrecisionSpec.fp16, "fp32": core.PrecisionSpec.fp32,
        "fp64": core.PrecisionSpec.fp64}


def same(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


# ------------------------------------------------------------------ CPU
def test_reference_api_surface():
    names = ["Format", "AccumKind", "AccumStrategy", "EmaxModel", "PrecisionSpec", "quantize", "Matrix",
             "gemm_emulated", "gemm_emulated_with_accum", "accumulates_in_float", "reduce_in_precision",
             "VerifyMode", "checksum_precision_for", "ChecksumVectors", "EncodedProduct", "encode_and_multiply",
             "row_sums", "RowStats", "row_stats", "VabftParams", "ThresholdBreakdown", "precompute_b_stats",
             "BStatsSummary", "threshold_row", "resolve_e_max", "vabft_thresholds", "AabftParams", "aabft_sigma",
             "AabftThresholds", "aabft_threshold", "aabft_computed_y", "RowVerdict", "DetectOptions", "localize",
             "verify", "correct", "Philox", "Distribution", "random_matrix", "FaultTarget", "FlipDirection",
             "FaultSpec", "InjectionRecord", "encode_bits", "decode_bits", "inject", "CampaignConfig",
             "CampaignOutcome", "injection_campaign"]
    missing = [n for n in names if not hasattr(core, n)]
    assert not missing, missing


def test_philox_streams_match_reference(ref_or_port):
    for seed, stream in [(0, 0), (12345, 7), (2 ** 40 + 3, 2 ** 33)]:
        p = core.Philox(seed, stream)
        assert [p.next_u32() for _ in range(41)] == list(ref_or_port.draws(seed, stream, 0, 41))
        p = core.Philox(seed, stream)
        assert [p.next_u64() for _ in range(9)] == list(ref_or_port.draws(seed, stream, 1, 9))
        p = core.Philox(seed, stream)
        assert same([p.next_double() for _ in range(17)], ref_or_port.draws(seed, stream, 2, 17))
        p = core.Philox(seed, stream)
        assert same([p.normal() for _ in range(2000)], ref_or_port.draws(seed, stream, 3, 2000))
        p = core.Philox(seed, stream)
        assert [p.next_below(1000003) for _ in range(33)] == list(ref_or_port.draws(seed, stream, 4, 33, 1000003))
    # Philox KAT (proj/tests/unit/test_rng.cpp:9-21 uses the published vectors)
    assert core.Philox.block([0, 0, 0, 0], [0, 0]) == ref_or_port.philox_block([0, 0, 0, 0], [0, 0])


@pytest.mark.parametrize("fmt", list(FMTS))
@pytest.mark.parametrize("dist", ["normal:0,1", "normal:1e-6,1", "uniform:-1,1", "truncnormal:0,1,-1,1", "absnormal:1,1"])
def test_random_matrix_matches_reference(ref_or_port, fmt, dist):
    A, B = ref_or_port.trial_inputs(7, 13, 5, fmt, dist, 99, 3)
    rng = core.Philox(99, 3)
    d = core.Distribution.parse(dist)
    a = core.random_matrix(7, 13, d, SPEC[fmt](), rng)
    b = core.random_matrix(13, 5, d, SPEC[fmt](), rng)
    assert same(a.values(), A) and same(b.values(), B)


def test_host_scalars_match_reference(ref_or_port, golden):
    for fmt in FMTS:
        spec = SPEC[fmt]()
        for x in [0.0, 1.0, -3.14159, 1e-30, 65519.0, 1e38, 2.0 ** -140, 123456.789]:
            assert same(core.quantize(x, spec), ref_or_port.quantize(x, fmt))
            v = ref_or_port.quantize(x, fmt)
            assert core.encode_bits(v, FMTS[fmt]) == ref_or_port.encode_bits(v, fmt)
            b = ref_or_port.encode_bits(v, fmt)
            assert same(core.decode_bits(b, FMTS[fmt]), ref_or_port.decode_bits(b, fmt))
    for d1, d2, n in [(1.0, 6.0, 10), (2.0, 12.0, 10), (0.0, 1.0, 4), (1e-300, 5.0, 3), (3.0, float("nan"), 5),
                      (1.0, 2.5, 8), (-2.0, -7.0, 100)]:
        assert core.localize(d1, d2, n) == ref_or_port.localize(d1, d2, n)
    for n, t, y in [(128, 8, 3.5), (4096, 23, 21.0), (1, 53, 1.0)]:
        assert core.aabft_sigma(n, t, y) == ref_or_port.aabft_sigma(n, t, y)
    for fmt in FMTS:
        for dim in (1, 256, 4096):
            assert core.resolve_e_max(SPEC[fmt](), dim) == ref_or_port.resolve_e_max(fmt, dim)


def test_threshold_row_hand_case():
    # proj/tests/unit/test_threshold_vabft.cpp:11-27 style hand case, checked
    # against the formula of threshold_vabft.cpp:28-42 written out here
    a = core.RowStats()
    a.mean, a.max, a.min, a.var_bound, a.n = 0.5, 1.0, 0.0, 0.25, 4
    b = core.BStatsSummary()
    b.sum_abs_mean, b.sum_mean_sq, b.sum_var, b.k_len = 2.0, 1.5, 0.5, 4
    t = core.threshold_row(a, b, 3, core.VabftParams(1e-3, 2.5))
    det = 3 * 0.5 * 2.0
    var23 = 2.5 * math.sqrt(3 * 0.25 * 0.5 + 9 * 0.25 * 1.5)
    var4 = 2.5 * math.sqrt(3) * 0.5 * math.sqrt(0.5)
    assert (t.det, t.var23, t.var4) == (det, var23, var4)
    assert t.total == 1e-3 * (det + var23 + var4)
    s = core.BStatsSummary.from_([a, a])
    assert (s.sum_abs_mean, s.sum_mean_sq, s.sum_var, s.k_len) == (1.0, 0.5, 0.5, 2)
    bad = core.RowStats()
    bad.var_bound = -1.0
    with pytest.raises(RuntimeError):  # std::logic_error
        core.BStatsSummary.from_([bad])
    with pytest.raises(ValueError):
        core.BStatsSummary.from_([])


@pytest.mark.parametrize("fmt,bit,src32", [("bf16", 9, False), ("fp16", 14, False), ("fp32", 27, False),
                                           ("bf16", 30, True), ("fp64", 60, False)])
@pytest.mark.parametrize("direction", [0, 1, 2, 3])
def test_inject_matches_reference(ref_or_port, fmt, bit, src32, direction):
    X, _ = ref_or_port.trial_inputs(9, 11, 1, "fp32" if src32 else fmt, "normal:1e-6,1", 5, 1)
    spec = core.PrecisionSpec.fp32() if src32 else SPEC[fmt]()
    m = core.Matrix.from_numpy(X, spec, False)
    for seed, pos in [(3, None), (4, None), (5, (2, 7)), (6, (8, 10))]:
        Xr, rec = ref_or_port.inject(X, fmt, bit, direction=direction, pos=pos, seed=seed, stream=2, src_fp32=src32)
        f = core.FaultSpec()
        f.bit_index, f.direction = bit, core.FlipDirection(direction)
        if pos is not None:
            f.position = pos
        out, r = core.inject(m, f, core.Philox(seed, 2))
        assert (r.i, r.j, r.applied, int(r.direction_taken)) == (rec["i"], rec["j"], rec["applied"], rec["direction_taken"])
        assert same(out.values(), Xr)
        assert same([r.value_before, r.value_after], [rec["value_before"], rec["value_after"]])
    with pytest.raises(IndexError):  # std::out_of_range
        f = core.FaultSpec()
        f.bit_index = 64
        core.inject(m, f, core.Philox(0))


def test_matrix_semantics():
    s = core.PrecisionSpec.bf16()
    m = core.Matrix.from_numpy(np.array([[1.0, 1.00390625], [3.0, -2.5]]), s)
    assert m.values()[0, 1] == 1.0  # RNE to bf16
    with pytest.raises(ValueError):
        core.Matrix.from_numpy(np.array([[1.00390625]]), s, False)
    with pytest.raises(IndexError):
        m.at(2, 0)
    with pytest.raises(ValueError):  # quantize: non-finite input is a domain_error
        m.set(0, 0, float("inf"))
    m2 = core.Matrix.identity(2, s)
    assert m2.values().tolist() == [[1.0, 0.0], [0.0, 1.0]] and not m2.same_bits(m)
    assert core.checksum_precision_for(s, core.VerifyMode.Online).format == core.Format.FP32
    with pytest.raises(ValueError):
        core.ChecksumVectors.make(2 ** 24 + 1, core.PrecisionSpec.fp32())


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU behaviour")
def test_device_entry_points_fail_loudly_without_gpu():
    s = core.PrecisionSpec.bf16()
    a = core.Matrix.from_numpy(np.ones((2, 3)), s)
    b = core.Matrix.from_numpy(np.ones((3, 2)), s)
    with pytest.raises(RuntimeError):  # vabft.device_error: no CPU fallback
        core.encode_and_multiply(a, b)
    with pytest.raises(RuntimeError):
        core.row_stats(np.ones(4))


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("fmt", list(FMTS))
@pytest.mark.parametrize("mode", ["offline", "online"])
def test_encode_verify_correct_bit_exact(ref_or_port, fmt, mode):
    A, B = ref_or_port.trial_inputs(24, 200, 40, fmt, "normal:1e-6,1", 17, 4)
    s = SPEC[fmt]()
    a, b = core.Matrix.from_numpy(A, s, False), core.Matrix.from_numpy(B, s, False)
    vm = core.VerifyMode.Online if mode == "online" else core.VerifyMode.Offline
    e = core.encode_and_multiply(a, b, vm)
    r = ref_or_port.encode_and_multiply(A, B, fmt, mode)
    assert same(e.c.values(), r.c) and same(e.c_accum.values(), r.c_accum)
    for x, y in [(e.row_check1, r.row_check1), (e.row_check2, r.row_check2), (e.col_check1, r.col_check1),
                 (e.col_check2, r.col_check2)]:
        assert same(x, y)
    g = core.gemm_emulated_with_accum(a, b)
    assert same(g.c.values(), r.c) and same(g.accum.values(), r.c_accum)
    # statistics and thresholds
    T = core.vabft_thresholds(a, b, core.VabftParams(8e-3, 2.5))
    Tr, bsum = ref_or_port.vabft_thresholds(A, B, 8e-3, 2.5, fmt)
    assert same(T, Tr)
    bs = core.precompute_b_stats(b)
    s_ = core.BStatsSummary.from_(bs)
    assert same([s_.sum_abs_mean, s_.sum_mean_sq, s_.sum_var], bsum[:3])
    st = core.row_stats(A[3])
    rs = ref_or_port.row_stats(A[3])
    assert same([st.mean, st.max, st.min, st.var_bound], rs[:4])
    # row sums in the checksum precision, then verify with one injected fault
    src = e.verification_source()
    r1, r2 = core.row_sums(src, e.checksum_precision)
    q1, q2 = ref_or_port.row_sums(r.c_accum if mode == "online" else r.c, fmt, mode)
    assert same(r1, q1) and same(r2, q2)
    f = core.FaultSpec()
    f.bit_index, f.direction, f.position = (28 if mode == "online" or fmt in ("fp32",) else (60 if fmt == "fp64" else 13)), \
        core.FlipDirection.Flip, (5, 17)
    if mode == "online":
        bad, rec = core.inject(e.c_accum, f, core.Philox(1))
        e.c_accum = bad
    else:
        bad, rec = core.inject(e.c, f, core.Philox(1))
        e.c = bad
    v = core.verify(e, T)
    vr = ref_or_port.verify(bad.values(), r.row_check1, r.row_check2, Tr, fmt, mode)
    assert same([x.diff1 for x in v], vr["diff1"]) and same([x.diff2 for x in v], vr["diff2"])
    assert [x.detected for x in v] == list(vr["detected"].astype(bool))
    assert [(-1 if x.location is None else x.location) for x in v] == list(vr["location"])
    if v[5].detected and v[5].location is not None and mode == "offline":
        fixed = core.correct(e.c, v[5])
        assert fixed.rows() == e.c.rows()


@pytest.mark.gpu
def test_aabft_computed_y_bit_exact(ref_or_port):
    A, B = ref_or_port.trial_inputs(8, 64, 48, "bf16", "normal:0,1", 3, 0)
    s = core.PrecisionSpec.bf16()
    a, b = core.Matrix.from_numpy(A, s, False), core.Matrix.from_numpy(B, s, False)
    p = core.AabftParams.for_format(core.Format.BF16)
    t = core.aabft_threshold(a, b, p)
    tr = ref_or_port.aabft_threshold(A, B, "bf16")
    assert same(t.per_row, tr[0]) and t.y_used == tr[1]


@pytest.mark.gpu
@pytest.mark.parametrize("mode,bit", [("offline", 10), ("online", 20)])
def test_injection_campaign_counts_equal_reference(ref_or_port, mode, bit):
    cfg = core.CampaignConfig()
    cfg.m, cfg.k, cfg.n = 16, 64, 24
    cfg.precision = core.PrecisionSpec.bf16()
    cfg.dist = core.Distribution.parse("normal:1e-6,1")
    cfg.bit_index, cfg.trials, cfg.seed = bit, 12, 21
    cfg.mode = core.VerifyMode.Online if mode == "online" else core.VerifyMode.Offline
    cfg.direction = core.FlipDirection.Set0To1
    e_max = 8e-3 if mode == "offline" else 4e-6
    out = core.injection_campaign(cfg, lambda a, b: core.vabft_thresholds(a, b, core.VabftParams(e_max, 2.5)))
    tot = np.zeros(4, dtype=np.int64)
    for trial in range(cfg.trials):
        o = ref_or_port.campaign_trial(16, 64, 24, "bf16", "normal:1e-6,1", bit, 21, trial, mode=mode, method=0,
                                       e_max=e_max)
        tot += o[:4]
    assert (out.applicable, out.detected, out.located_correctly, out.nonfinite_after) == tuple(int(x) for x in tot)


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["bf16", "fp32", "fp64"])
def test_cpp_fused_gemm_matches_python_path(fmt):
    """vabft::b200::FusedGemm (the C++ drop-in's hot path) == FusedAbftGemm
    on the same device inputs: C, thresholds, verdicts bit-identical."""
    import torch
    from paper_2602_08043_b200 import _core
    from paper_2602_08043_b200.fused import FusedAbftGemm
    dt = {"bf16": torch.bfloat16, "fp32": torch.float32, "fp64": torch.float64}[fmt]
    torch.manual_seed(5)
    m, k, n = 256, 512, 384
    A = torch.randn(m, k, device="cuda").to(dt)
    B = torch.randn(k, n, device="cuda").to(dt)
    py = FusedAbftGemm(B, mode="online")
    r = py(A)
    F = {"bf16": _core.Format.BF16, "fp32": _core.Format.FP32, "fp64": _core.Format.FP64}[fmt]
    g = _core.FusedGemm(F, _core.VerifyMode.Online, k, n, B.data_ptr(), py.opts.e_max,
                        torch.cuda.current_stream().cuda_stream)
    C = torch.empty(m, n, device="cuda", dtype=dt)
    T = torch.empty(m, device="cuda", dtype=torch.float64)
    det = torch.empty(m, device="cuda", dtype=torch.uint8)
    loc = torch.empty(m, device="cuda", dtype=torch.int64)
    counts = torch.zeros(6, device="cuda", dtype=torch.int64)
    g(m, A.data_ptr(), C.data_ptr(), T.data_ptr(), det.data_ptr(), loc.data_ptr(), counts.data_ptr(),
      torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(C.view(torch.uint8), r.C.view(torch.uint8))
    assert torch.equal(T, r.T) and torch.equal(det, r.detected) and torch.equal(loc, r.location)
    assert int(counts[0]) == m and int(counts[1]) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", list(FMTS))
@pytest.mark.parametrize("mode", ["offline", "online"])
def test_reference_signature_reaches_the_fast_path(ref_or_port, fmt, mode):
    """b200::set_engine(Tensor): the reference-signature encode_and_multiply
    runs the B200 kernels (tcgen05 / 3xTF32 / DFMA). C_accum is the tensor
    core's, within the FP32-accumulate bound of the exact product; the
    checksums are the fused path's (working type, NativeBlocked(128)) and
    equal the reference's row_sums composition bit for bit; verify() on the
    product flags and locates a planted fault exactly as the reference's
    verify does on the same data."""
    A, B = ref_or_port.trial_inputs(64, 256, 96, fmt, "normal:0,1", 23, 1)
    s = SPEC[fmt]()
    a, b = core.Matrix.from_numpy(A, s, False), core.Matrix.from_numpy(B, s, False)
    vm = core.VerifyMode.Online if mode == "online" else core.VerifyMode.Offline
    core.set_engine(core.Engine.Tensor)
    try:
        e = core.encode_and_multiply(a, b, vm)
    finally:
        core.set_engine(core.Engine.Exact)
    assert core.engine() == core.Engine.Exact
    exact = A @ B
    bound = (A.shape[1] + 1) * 2.0**-24 * (np.abs(A) @ np.abs(B))
    assert np.all(np.abs(e.c_accum.values() - exact) <= bound)
    c1, c2 = ref_or_port.blocked_row_checksums(A, B, fmt, mode)
    assert same(e.row_check1, c1) and same(e.row_check2, c2)
    T = np.full(A.shape[0], 1e-2 if fmt in ("bf16", "fp16") else 1e-6)
    f = core.FaultSpec()
    f.bit_index = 60 if fmt == "fp64" else (28 if (mode == "online" or fmt == "fp32") else 13)
    f.direction, f.position = core.FlipDirection.Flip, (7, 33)
    src = e.c_accum if mode == "online" else e.c
    bad, rec = core.inject(src, f, core.Philox(3))
    if mode == "online":
        e.c_accum = bad
    else:
        e.c = bad
    v = core.verify(e, T)
    wf = "fp64" if fmt == "fp64" else "fp32"
    vr = ref_or_port.verify(bad.values(), e.row_check1, e.row_check2, T, wf, "offline", accum=(2, 128))
    assert [x.detected for x in v] == list(vr["detected"].astype(bool))
    assert [(-1 if x.location is None else x.location) for x in v] == list(vr["location"])
    assert v[7].detected and v[7].location == 33
