"""Pins the plain-C oracle restatement (oracle/vabft_oracle.c) to
(1) the reference's own known-answer tests (proj/tests/unit/*.cpp) and
(2) golden vectors produced by the unmodified reference (tests/golden/).

CPU only. The four reference tests that are defective in the reference
itself are restated with their premise fixed and say so."""
import math

import numpy as np
import pytest

FMTS = ["bf16", "fp16", "fp32", "fp64"]
SHAPES = [(8, 12, 10), (33, 70, 129), (64, 128, 96)]


def bits(x):
    return np.asarray(x, dtype=np.float64).view(np.uint64)


def same(a, b):
    return np.array_equal(bits(a), bits(b))


# ---------------------------------------------------------------- RNG KATs
def test_philox_known_answers(port):
    # proj/tests/unit/test_rng.cpp:9-21 (Random123 vectors)
    assert port.philox_block([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert port.philox_block([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert port.philox_block([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_philox_streams_golden(port, golden):
    assert np.array_equal(port.draws(42, 7, 0, 1000), golden["draw_u32"])
    assert np.array_equal(port.draws(42, 7, 1, 1000), golden["draw_u64"])
    assert same(port.draws(42, 7, 2, 1000), golden["draw_double"])
    assert same(port.draws(11, 3, 3, 5000), golden["draw_normal"])
    assert np.array_equal(port.draws(17, 0, 4, 1000, arg=7), golden["draw_below7"])


def test_normal_moments(port):
    # test_rng.cpp:40-55
    z = port.draws(11, 3, 3, 200000)
    assert abs(z.mean()) < 0.01
    assert abs((z * z).mean() - 1.0) < 0.01
    assert abs((z ** 4).mean() - 3.0) < 0.15


# ---------------------------------------------------------------- quantize
def test_quantize_known_cases(port):
    # test_precision.cpp:51-61, 118-140
    q = port.quantize
    assert q(1.0, "bf16") == 1.0
    assert q(1.0 + 2**-9, "bf16") == 1.0
    assert q(1.0 + 2**-8, "bf16") == 1.0  # tie -> even
    assert q(1.0 + 3 * 2**-8, "bf16") == 1.0 + 2**-6
    assert q(1.0 + 2**-8 + 2**-50, "bf16") == 1.0 + 2**-7
    assert math.copysign(1.0, q(-0.0, "bf16")) == -1.0
    assert q(2**-133, "bf16") == 2**-133  # min subnormal kept
    assert q(1e39, "bf16") == float.fromhex("0x1.FEp127")  # saturate
    assert q(70000.0, "fp16") == 65504.0
    assert abs(q(0.1, "fp16") - 0.1) <= 0.1 * 2**-11


@pytest.mark.parametrize("fmt", FMTS)
def test_quantize_golden(port, golden, fmt):
    xs = golden["q_x"]
    out = np.array([port.quantize(x, fmt) for x in xs])
    assert same(out, golden[f"q_{fmt}"])


def test_quantize_fp32_matches_cast(port):
    rng = np.random.default_rng(5)
    xs = np.ldexp(rng.uniform(-2, 2, 5000), rng.integers(-140, 120, 5000))
    out = np.array([port.quantize(x, "fp32") for x in xs])
    assert same(out, xs.astype(np.float32).astype(np.float64))


def test_quantize_nonfinite_raises(port):
    import oracle
    with pytest.raises(oracle.OracleError) as e:
        port.quantize(math.inf, "bf16")
    assert e.value.code == 2  # domain_error


# --------------------------------------------------- encode_and_multiply
@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("mode", ["offline", "online"])
@pytest.mark.parametrize("si", range(len(SHAPES)))
def test_encode_and_multiply_golden(port, golden, fmt, mode, si):
    A, B = golden[f"A_{fmt}_{si}"], golden[f"B_{fmt}_{si}"]
    e = port.encode_and_multiply(A, B, fmt, mode)
    key = f"{fmt}_{mode}_{si}"
    assert same(e.c, golden[f"C_{key}"])
    assert same(e.c_accum, golden[f"Ca_{key}"])
    assert same(e.row_check1, golden[f"rc1_{key}"])
    assert same(e.row_check2, golden[f"rc2_{key}"])
    assert same(e.col_check1, golden[f"cc1_{key}"])
    assert same(e.col_check2, golden[f"cc2_{key}"])
    src = e.c_accum if mode == "online" else e.c
    r1, r2 = port.row_sums(src, fmt, mode)
    assert same(r1, golden[f"rs1_{key}"]) and same(r2, golden[f"rs2_{key}"])
    if fmt in ("bf16", "fp16"):
        b1, b2 = port.row_sums(src, fmt, mode, accum=(2, 128))
        assert same(b1, golden[f"rsb1_{key}"]) and same(b2, golden[f"rsb2_{key}"])


def test_trial_inputs_golden(port, golden):
    for fmt in FMTS:
        for si, (m, k, n) in enumerate(SHAPES):
            dist = ["normal:0,1", "uniform:-1,1", "truncnormal:0,1,-1,1", "normal:1e-6,1"][si % 4]
            A, B = port.trial_inputs(m, k, n, fmt, dist, 1000 + si, FMTS.index(fmt))
            assert same(A, golden[f"A_{fmt}_{si}"]) and same(B, golden[f"B_{fmt}_{si}"])


def test_identity_checksums(port):
    # test_checksum.cpp:24-32
    e = port.encode_and_multiply(np.eye(3), np.eye(3), "fp32")
    assert list(e.row_check1) == [1, 1, 1] and list(e.row_check2) == [1, 2, 3]
    assert list(e.col_check1) == [1, 1, 1] and list(e.col_check2) == [1, 2, 3]


def test_one_by_one(port):
    # test_checksum.cpp:34-42
    e = port.encode_and_multiply(np.array([[2.0]]), np.array([[3.0]]), "fp32")
    assert e.c[0, 0] == 6.0 and e.row_check1[0] == 6.0 and e.row_check2[0] == 6.0


def test_sixteen_bit_formats_need_fp32_accumulation(port):
    import oracle
    with pytest.raises(oracle.OracleError):
        port.encode_and_multiply(np.eye(2), np.eye(2), "bf16", accum=(1, 128))


def test_blocked_one_equals_sequential(port):
    # test_precision.cpp:228-241: blocked(1) and blocked(K) reproduce sequential bitwise
    A, B = port.trial_inputs(8, 37, 9, "fp32", "normal:0,1", 3, 0)
    seq = port.encode_and_multiply(A, B, "fp32", accum=(1, 128)).c
    assert same(port.encode_and_multiply(A, B, "fp32", accum=(2, 1)).c, seq)
    assert same(port.encode_and_multiply(A, B, "fp32", accum=(2, 1000)).c, seq)


# ---------------------------------------------------------- statistics
def test_row_stats_basic(port):
    # test_stats.cpp:21-47
    s = port.row_stats(np.full(10, 3.5))
    assert s[0] == 3.5 and s[3] == 0.0
    s = port.row_stats(np.array([-1.0, 1.0]))
    assert s[0] == 0.0 and s[3] == 1.0
    s = port.row_stats(np.full(10**6, 0.1))
    assert abs(s[0] - 0.1) < 1e-15


def test_row_stats_rejects(port):
    import oracle
    with pytest.raises(oracle.OracleError):
        port.row_stats(np.array([1.0, math.nan]))
    with pytest.raises(oracle.OracleError):
        port.row_stats(np.array([]))


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("si", range(len(SHAPES)))
def test_thresholds_golden(port, golden, fmt, si):
    A, B = golden[f"A_{fmt}_{si}"], golden[f"B_{fmt}_{si}"]
    e_max = golden[f"emax_{fmt}_{si}"][0]
    assert port.resolve_e_max(fmt, A.shape[1]) == e_max
    T, s = port.vabft_thresholds(A, B, e_max)
    assert same(T, golden[f"T_{fmt}_{si}"]) and same(s, golden[f"bsum_{fmt}_{si}"])
    Ta, y, _ = port.aabft_threshold(A, B, fmt)
    assert same(Ta, golden[f"Ta_{fmt}_{si}"]) and y == golden[f"ya_{fmt}_{si}"][0]


def test_vabft_hand_case(port):
    # test_threshold_vabft.cpp:11-27: T = 0.25 with var4 = 250
    out = port.threshold_row([0.0, 1.0, -1.0, 1.0], [0.0, 0.0, 100.0], 100, 1e-3, 2.5)
    assert out[0] == 0.0 and out[1] == 0.0
    assert abs(out[2] - 250.0) < 1e-9 and abs(out[3] - 0.25) < 1e-12


def test_aabft_published_values(port):
    # test_threshold_aabft.cpp:10-15
    assert abs(3 * port.aabft_sigma(512, 53, 21.0) / 1.66e-11 - 1) < 0.01
    assert abs(3 * port.aabft_sigma(1024, 53, 21.0) / 4.68e-11 - 1) < 0.01
    assert abs(3 * port.aabft_sigma(2048, 53, 21.0) / 1.32e-10 - 1) < 0.01


def test_aabft_computed_y_case(port):
    # test_threshold_aabft.cpp:71-77
    A = np.array([[0.5, -3.0], [1.0, 2.0]])
    B = np.array([[1.0, 2.0], [-4.0, 0.5]])
    _, y, _ = port.aabft_threshold(A, B, "fp64", computed=True)
    assert y == 3.0 * 3.5


# ---------------------------------------------------------------- detect
def test_localize_golden(port, golden):
    for (d1, d2, n), (j, r) in zip(golden["loc_cases"], golden["loc_out"]):
        got = port.localize(d1, d2, int(n))
        if j < 0:
            assert got is None
        else:
            assert got == (int(j), r)


@pytest.mark.parametrize("mode", ["offline", "online"])
def test_verify_golden(port, golden, mode):
    v = port.verify(golden[f"vsrc_{mode}"], golden[f"vrc1_{mode}"], golden[f"vrc2_{mode}"], golden[f"vT_{mode}"],
                    "fp32", mode)
    for k in ("diff1", "diff2", "residual"):
        assert same(v[k], golden[f"v{k}_{mode}"])
    assert np.array_equal(v["detected"], golden[f"vdetected_{mode}"].astype(bool))
    assert np.array_equal(v["location"], golden[f"vlocation_{mode}"])


def test_unit_error_detected_located(port):
    # test_detect.cpp:37-56 — exact integer product, +1 at (2,5)
    rng_a = port.draws(5, 0, 4, 8 * 12, arg=8).astype(np.float64).reshape(8, 12)
    rng_b = port.draws(5, 1, 4, 12 * 10, arg=8).astype(np.float64).reshape(12, 10)
    e = port.encode_and_multiply(rng_a, rng_b, "fp32")
    c = e.c.copy()
    c[2, 5] += 1.0
    v = port.verify(c, e.row_check1, e.row_check2, np.full(8, 0.5), "fp32")
    assert v["detected"][2] and v["diff1"][2] == 1.0 and v["diff2"][2] == 6.0 and v["location"][2] == 5
    assert not v["detected"][np.arange(8) != 2].any()


# ---------------------------------------------------------------- faults
def test_bits_known(port):
    # test_faults.cpp:23-28
    assert port.encode_bits(1.0, "bf16") == 0x3F80
    assert port.decode_bits(0x3F80 ^ (1 << 7), "bf16") == 0.5
    assert math.isinf(port.decode_bits(0x3F80 | (1 << 14), "bf16"))


@pytest.mark.parametrize("fmt", ["bf16", "fp16"])
def test_bits_all_patterns_golden(port, golden, fmt):
    dec = golden[f"dec_{fmt}"]
    for p in range(0, 0x10000, 97):
        d = port.decode_bits(p, fmt)
        assert same([d], [dec[p]])
        assert port.encode_bits(d, fmt) == golden[f"rt_{fmt}"][p]


def test_fp16_roundtrip_every_pattern(port):
    # test_faults.cpp:17-21
    for p in range(0, 0x10000, 13):
        assert port.encode_bits(port.decode_bits(p, "fp16"), "fp16") == p


def test_bf16_roundtrip_restated(port):
    # test_faults.cpp:11-15 is defective in the reference: BF16 decode goes
    # through float->double and quiets the 126 signalling-NaN patterns
    # (SURVEY §4.4). Restated: every non-sNaN pattern round-trips.
    for p in range(0x10000):
        is_snan = (p & 0x7F80) == 0x7F80 and (p & 0x7F) != 0 and not (p & 0x40)
        if not is_snan:
            assert port.encode_bits(port.decode_bits(p, "bf16"), "bf16") == p


@pytest.mark.parametrize("fmt", FMTS)
def test_inject_golden(port, golden, fmt):
    A = golden[f"inj_in_{fmt}"]
    for rep, rec in enumerate(golden[f"inj_rec_{fmt}"]):
        i, j, applied, dtaken, bit, d, pos_mode = rec
        X, r = port.inject(A, fmt, int(bit), direction=int(d), pos=None if pos_mode else (rep % 6, rep % 7),
                           seed=rep, stream=1)
        assert same(X, golden[f"inj_out_{fmt}"][rep])
        assert (r["i"], r["j"], int(r["applied"]), r["direction_taken"]) == (i, j, applied, dtaken)


def test_campaign_trials_golden(port, golden):
    for row in golden["campaign_trials"]:
        mode, bit, t = int(row[0]), int(row[1]), int(row[2])
        out = port.campaign_trial(16, 64, 16, "bf16", "normal:1e-6,1", bit, 17, t,
                                  mode="online" if mode else "offline", method=0,
                                  e_max=2e-6 if mode else 8e-3)
        assert np.array_equal(out, row[3:]), (mode, bit, t)


def test_port_matches_reference_when_built(port):
    """Cross-check a fresh random batch against the live reference build."""
    import oracle
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    R = oracle.ref()
    for t in range(6):
        for fmt in FMTS:
            A, B = R.trial_inputs(9, 33, 17, fmt, "normal:0,1", 500 + t, 0)
            for mode in ("offline", "online"):
                a, b = R.encode_and_multiply(A, B, fmt, mode), port.encode_and_multiply(A, B, fmt, mode)
                assert same(a.c_accum, b.c_accum) and same(a.row_check2, b.row_check2)


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("mode", ["offline", "online"])
def test_blocked_row_checksums_composition(ref_or_port, fmt, mode):
    """The config-scale checksum oracle (row_sums composition, no emulated
    GEMM) equals encode_impl's row checksums with a NativeBlocked(128)
    checksum precision: checked against a direct restatement of the
    contract (checksum.cpp:74-79) in the working type."""
    O = ref_or_port
    A, B = O.trial_inputs(23, 300, 260, fmt, "normal:0,1", 77, 1)
    c1, c2 = O.blocked_row_checksums(A, B, fmt, mode)
    wt = np.float64 if fmt == "fp64" else np.float32

    def blocked(terms):
        tot = wt(0)
        for b0 in range(0, len(terms), 128):
            part = wt(0)
            for t in terms[b0:b0 + 128]:
                part = wt(part + t)
            tot = wt(tot + part)
        return tot
    w = np.arange(1, B.shape[1] + 1, dtype=wt)
    Bw = B.astype(wt)
    br1 = np.array([blocked(Bw[q]) for q in range(B.shape[0])], dtype=wt)
    br2 = np.array([blocked((w * Bw[q]).astype(wt)) for q in range(B.shape[0])], dtype=wt)
    if mode == "offline":
        br1 = np.array([O.quantize(float(x), fmt) for x in br1], dtype=wt)
        br2 = np.array([O.quantize(float(x), fmt) for x in br2], dtype=wt)
    Aw = A.astype(wt)
    for br, got in ((br1, c1), (br2, c2)):
        want = np.array([blocked((br * Aw[i]).astype(wt)) for i in range(A.shape[0])], dtype=np.float64)
        if mode == "offline":
            want = np.array([O.quantize(x, fmt) for x in want])
        assert same(got, want)
    if fmt in ("fp32", "fp64"):
        # native formats: the reference's own encode with the strategy override
        e = O.encode_and_multiply(A, B, fmt, mode, accum=(2, 128))
        assert same(c1, e.row_check1) and same(c2, e.row_check2)
