"""GPU parity of the wide-format fused path (K5: FP64 SIMT DFMA GEMM + the
shared verify tail) against the oracle.

Bars: C within the FP64 accumulation bound (test_precision.cpp:181-206 with
u = 2^-53); checksums, row sums, thresholds, verdicts, locations and counts
bit-exact against the oracle run on the device's own C with an FP64
NativeBlocked(128) checksum precision (the TENSOR engine's).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BLK = (2, 128)  # AccumKind::NativeBlocked, block 128


def bits(x):
    return np.asarray(x, dtype=np.float64).view(np.uint64)


def same(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    na, nb = np.isnan(a), np.isnan(b)
    return a.shape == b.shape and np.array_equal(na, nb) and np.array_equal(bits(a[~na]), bits(b[~nb]))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.mark.parametrize("mode", ["offline", "online"])
@pytest.mark.parametrize("shape", [(64, 128, 96), (200, 264, 72), (256, 520, 384)])
def test_fp64_tensor_engine_parity(torch_cuda, port, mode, shape):
    from paper_2602_08043_b200 import api
    m, k, n = shape
    A, B = port.trial_inputs(m, k, n, "fp64", "normal:0,1", 5, 1)
    e = api.encode_and_multiply(A, B, mode, "fp64", engine="tensor")
    o = port.encode_and_multiply(A, B, "fp64", mode, accum=BLK)
    bound = 2 * (k + 1) * 2.0**-53 * (np.abs(A) @ np.abs(B))
    assert np.all(np.abs(e.c - o.c) <= bound)
    assert same(e.c, e.c_accum)
    assert same(e.row_check1, o.row_check1) and same(e.row_check2, o.row_check2)
    r1, r2 = api.row_sums(e.c, e.checksum_precision, "fp64")
    p1, p2 = port.row_sums(e.c, "fp64", "offline", accum=BLK)
    assert same(r1, p1) and same(r2, p2)


def _fused(torch, A, B, mode, **kw):
    from paper_2602_08043_b200.fused import FusedAbftGemm
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    return FusedAbftGemm(dB, mode=mode, **kw), dA


@pytest.mark.parametrize("mode", ["online", "offline"])
@pytest.mark.parametrize("bit", [2, 30, 51, 62])
def test_fp64_fused_injection_matches_oracle(torch_cuda, port, mode, bit):
    torch = torch_cuda
    from paper_2602_08043_b200 import api
    m, k, n = 160, 256, 392
    A, B = port.trial_inputs(m, k, n, "fp64", "normal:1e-6,1", 17, bit)
    cols = np.random.default_rng(bit).integers(0, n, m)
    e_max = 4e-15
    g, dA = _fused(torch, A, B, mode, e_max=e_max)
    rec = torch.zeros(m * 24, dtype=torch.uint8, device="cuda")
    f = {"col": torch.from_numpy(cols.astype(np.int32)).cuda(),
         "bit": torch.full((m,), bit, dtype=torch.int32, device="cuda"),
         "dir": torch.full((m,), 0, dtype=torch.int32, device="cuda"), "records": rec}
    counts = torch.zeros(6, dtype=torch.int64, device="cuda")
    r = g(dA, faults=f, checksums=True, counts=counts)
    torch.cuda.synchronize()
    Cf = r.C.cpu().numpy()
    # the clean product from the same kernel (TENSOR engine) and the flips
    e = api.encode_and_multiply(A, B, mode, "fp64", engine="tensor")
    flipped = e.c.copy()
    for i, j in enumerate(cols):
        flipped[i, j] = (np.array([e.c[i, j]]).view(np.uint64) ^ np.uint64(1 << bit)).view(np.float64)[0]
    assert same(Cf, flipped)
    applied = rec.view(m, 24)[:, 16:20].contiguous().view(torch.int32).view(m).cpu().numpy()
    assert np.all(applied == 1)  # Flip direction: always applicable
    # checksums and thresholds: bit-exact against the oracle
    o = port.encode_and_multiply(A, B, "fp64", mode, accum=BLK)
    assert same(r.row_check1.cpu().numpy(), o.row_check1) and same(r.row_check2.cpu().numpy(), o.row_check2)
    T_ref, _ = port.vabft_thresholds(A, B, e_max, fmt="fp64")
    assert same(r.T.cpu().numpy(), T_ref)
    # verdicts of the device's faulty C under the oracle's verify
    v = port.verify(Cf, o.row_check1, o.row_check2, T_ref, "fp64", mode, accum=BLK)
    assert np.array_equal(v["detected"], r.detected.cpu().numpy().astype(bool))
    assert np.array_equal(v["location"], r.location.cpu().numpy())
    assert same(v["diff1"], r.diff1.cpu().numpy()) and same(v["diff2"], r.diff2.cpu().numpy())
    c = counts.cpu().numpy()
    assert c[0] == m and c[1] == int(v["detected"].sum())
    if bit >= 51:  # high mantissa / exponent bits: every row caught
        assert v["detected"].all()
    if bit == 51:  # ... and located (at bit 62 the weighted sum overflows: no location, as in the reference)
        assert np.array_equal(v["location"], cols)


def test_fp64_fused_correction(torch_cuda, port):
    torch = torch_cuda
    m, k, n = 128, 192, 256
    A, B = port.trial_inputs(m, k, n, "fp64", "normal:0,1", 3, 0)
    g, dA = _fused(torch, A, B, "online", e_max=4e-15)
    clean = g(dA).C.clone()
    cols = (np.arange(m) * 7) % n
    f = {"col": torch.from_numpy(cols.astype(np.int32)).cuda(),
         "bit": torch.full((m,), 55, dtype=torch.int32, device="cuda"),
         "dir": torch.full((m,), 0, dtype=torch.int32, device="cuda")}
    counts = torch.zeros(6, dtype=torch.int64, device="cuda")
    r = g(dA, faults=f, counts=counts, correct=True)
    torch.cuda.synchronize()
    c = counts.cpu().numpy()
    assert c[1] == m and c[2] == m and c[5] == m
    err = (r.C - clean).abs().max().item() / clean.abs().max().item()
    assert err < 1e-12


@pytest.mark.parametrize("dist", ["normal:0,1", "uniform:-1,1", "truncnormal:0,1,-1,1"])
def test_fp64_fused_no_false_positives(torch_cuda, dist):
    torch = torch_cuda
    from paper_2602_08043_b200.campaign import sample_matrix
    from paper_2602_08043_b200.fused import FusedAbftGemm
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    for (m, k, n) in [(256, 1024, 512), (512, 4096, 256)]:
        A = sample_matrix((m, k), dist, gen, "cuda", torch.float64)
        B = sample_matrix((k, n), dist, gen, "cuda", torch.float64)
        counts = torch.zeros(6, dtype=torch.int64, device="cuda")
        for mode in ("online", "offline"):
            counts.zero_()
            FusedAbftGemm(B, mode=mode)(A, counts=counts)
            assert int(counts[1].item()) == 0, (dist, m, k, n, mode)


def test_fp64_plain_gemm_matches_torch(torch_cuda):
    torch = torch_cuda
    from paper_2602_08043_b200.fused import plain_gemm
    torch.manual_seed(0)
    for (m, n, k) in [(128, 128, 16), (200, 264, 72), (1000, 770, 514)]:
        a = torch.randn(m, k, device="cuda", dtype=torch.float64)
        b = torch.randn(k, n, device="cuda", dtype=torch.float64)
        c = plain_gemm(a, b)
        ref = a @ b
        bound = 2 * (k + 1) * 2.0**-53 * (a.abs() @ b.abs())
        assert bool(((c - ref).abs() <= bound).all())


# ---------------------------------------------------------------- FP32 (3xTF32)
def _prod_bound(A, B, k):
    """3xTF32 products (< 2^-21 relative each) accumulated in FP32 over k
    terms, against the oracle's FP32 pairwise product."""
    return (2 * (k + 1) * 2.0**-23 + 2.0**-20) * (np.abs(A) @ np.abs(B))


@pytest.mark.parametrize("mode", ["offline", "online"])
@pytest.mark.parametrize("shape", [(64, 128, 96), (200, 264, 72), (256, 520, 384)])
def test_fp32_tensor_engine_parity(torch_cuda, port, mode, shape):
    from paper_2602_08043_b200 import api
    m, k, n = shape
    A, B = port.trial_inputs(m, k, n, "fp32", "normal:0,1", 6, 1)
    e = api.encode_and_multiply(A, B, mode, "fp32", engine="tensor")
    o = port.encode_and_multiply(A, B, "fp32", mode, accum=BLK)
    assert np.all(np.abs(e.c - o.c) <= _prod_bound(A, B, k))
    assert same(e.c, e.c_accum)
    assert same(e.row_check1, o.row_check1) and same(e.row_check2, o.row_check2)
    r1, r2 = api.row_sums(e.c, e.checksum_precision, "fp32")
    p1, p2 = port.row_sums(e.c, "fp32", "offline", accum=BLK)
    assert same(r1, p1) and same(r2, p2)


@pytest.mark.parametrize("mode", ["online", "offline"])
@pytest.mark.parametrize("bit", [2, 15, 22, 30])
def test_fp32_fused_injection_matches_oracle(torch_cuda, port, mode, bit):
    torch = torch_cuda
    from paper_2602_08043_b200 import api
    m, k, n = 160, 256, 392
    A, B = port.trial_inputs(m, k, n, "fp32", "normal:1e-6,1", 23, bit)
    cols = np.random.default_rng(bit).integers(0, n, m)
    e_max = 2e-6
    from paper_2602_08043_b200.fused import FusedAbftGemm
    dA = torch.from_numpy(A).float().cuda()
    g = FusedAbftGemm(torch.from_numpy(B).float().cuda(), mode=mode, e_max=e_max)
    rec = torch.zeros(m * 24, dtype=torch.uint8, device="cuda")
    f = {"col": torch.from_numpy(cols.astype(np.int32)).cuda(),
         "bit": torch.full((m,), bit, dtype=torch.int32, device="cuda"),
         "dir": torch.full((m,), 0, dtype=torch.int32, device="cuda"), "records": rec}
    counts = torch.zeros(6, dtype=torch.int64, device="cuda")
    r = g(dA, faults=f, checksums=True, counts=counts)
    torch.cuda.synchronize()
    Cf = r.C.double().cpu().numpy()
    e = api.encode_and_multiply(A, B, mode, "fp32", engine="tensor")
    flipped = e.c.astype(np.float32)
    for i, j in enumerate(cols):
        flipped[i, j] = (np.array([flipped[i, j]], dtype=np.float32).view(np.uint32) ^ np.uint32(1 << bit)).view(
            np.float32)[0]
    assert same(Cf, flipped.astype(np.float64))
    o = port.encode_and_multiply(A, B, "fp32", mode, accum=BLK)
    assert same(r.row_check1.cpu().numpy(), o.row_check1) and same(r.row_check2.cpu().numpy(), o.row_check2)
    T_ref, _ = port.vabft_thresholds(A, B, e_max, fmt="fp32")
    assert same(r.T.cpu().numpy(), T_ref)
    v = port.verify(Cf, o.row_check1, o.row_check2, T_ref, "fp32", mode, accum=BLK)
    assert np.array_equal(v["detected"], r.detected.cpu().numpy().astype(bool))
    assert np.array_equal(v["location"], r.location.cpu().numpy())
    assert same(v["diff1"], r.diff1.cpu().numpy()) and same(v["diff2"], r.diff2.cpu().numpy())
    assert counts.cpu().numpy()[1] == int(v["detected"].sum())
    if bit in (22, 30):  # top mantissa / exponent bits: every row caught
        assert v["detected"].all()


def test_fp32_single_pass_tf32(torch_cuda):
    torch = torch_cuda
    from paper_2602_08043_b200.fused import FusedAbftGemm
    torch.manual_seed(3)
    m, k, n = 512, 1024, 768
    A = torch.randn(m, k, device="cuda")
    B = torch.randn(k, n, device="cuda")
    ref = A.double() @ B.double()
    g1 = FusedAbftGemm(B, tf32_passes=1, e_max=2e-3)
    g3 = FusedAbftGemm(B)
    c1 = torch.zeros(6, dtype=torch.int64, device="cuda")
    c3 = torch.zeros(6, dtype=torch.int64, device="cuda")
    r1 = g1(A, counts=c1)
    e1 = ((r1.C.double() - ref).abs().max() / ref.abs().max()).item()
    r3 = g3(A, counts=c3)
    e3 = ((r3.C.double() - ref).abs().max() / ref.abs().max()).item()
    assert e1 < 2e-3 and e3 < 1e-5 and e3 < e1 / 20, (e1, e3)
    assert int(c1[1]) == 0 and int(c3[1]) == 0


@pytest.mark.parametrize("dist", ["normal:0,1", "uniform:-1,1", "truncnormal:0,1,-1,1"])
def test_fp32_fused_no_false_positives(torch_cuda, dist):
    torch = torch_cuda
    from paper_2602_08043_b200.campaign import sample_matrix
    from paper_2602_08043_b200.fused import FusedAbftGemm
    gen = torch.Generator(device="cuda")
    gen.manual_seed(2)
    for (m, k, n) in [(256, 1024, 512), (512, 4096, 256)]:
        A = sample_matrix((m, k), dist, gen, "cuda", torch.float32)
        B = sample_matrix((k, n), dist, gen, "cuda", torch.float32)
        counts = torch.zeros(6, dtype=torch.int64, device="cuda")
        for mode in ("online", "offline"):
            counts.zero_()
            FusedAbftGemm(B, mode=mode)(A, counts=counts)
            assert int(counts[1].item()) == 0, (dist, m, k, n, mode)


def test_fp32_plain_gemm_matches_fp64(torch_cuda):
    torch = torch_cuda
    from paper_2602_08043_b200.fused import plain_gemm
    torch.manual_seed(0)
    for (m, n, k) in [(128, 256, 16), (200, 264, 72), (1000, 772, 516)]:
        a = torch.randn(m, k, device="cuda")
        b = torch.randn(k, n, device="cuda")
        c = plain_gemm(a, b)
        ref = a.double() @ b.double()
        bound = (2 * (k + 1) * 2.0**-23 + 2.0**-20) * (a.double().abs() @ b.double().abs())
        assert bool(((c.double() - ref).abs() <= bound).all())


def test_wide_rowstats_midpoint_fallback(torch_cuda, port):
    """Rows whose exact sum sits on a rounding midpoint take the reference's
    sequential Neumaier loop; every mean (hence T) stays bit-identical."""
    torch = torch_cuda
    from paper_2602_08043_b200.fused import FusedAbftGemm
    m, k, n = 32, 64, 64
    rng = np.random.default_rng(7)
    A = rng.standard_normal((m, k))
    A[0, :] = 0.0
    A[0, 0], A[0, 1] = 1.0, 2.0**-53          # 1 + 2^-53: exactly between 1 and 1 + 2^-52
    A[1, :] = 0.0
    A[1, 0], A[1, 5], A[1, 9] = 3.0, 2.0**-52, 2.0**-52 * 0.5
    A[2, :3] = [1e16, 1.0, -1e16]              # cancellation
    B = rng.standard_normal((k, n))
    counts = torch.zeros(6, dtype=torch.int64, device="cuda")
    g = FusedAbftGemm(torch.from_numpy(B).cuda(), e_max=4e-15)
    r = g(torch.from_numpy(A).cuda(), counts=counts)
    torch.cuda.synchronize()
    T_ref, _ = port.vabft_thresholds(A, B, 4e-15, fmt="fp64")
    assert same(r.T.cpu().numpy(), T_ref)
    assert int(counts[4].item()) >= 1  # the midpoint row went the sequential way


@pytest.mark.parametrize("fmt,target,bit", [("fp64", "A", 52), ("fp64", "B", 40), ("fp32", "A", 23),
                                            ("fp32", "B", 20)])
def test_wide_operand_faults_match_oracle(torch_cuda, port, fmt, target, bit):
    """Operand faults on the wide path: the GEMM multiplies the flipped operand,
    the checksums / thresholds come from the clean ones; verdicts bit-exact
    against the oracle's verify of the same product."""
    torch = torch_cuda
    from paper_2602_08043_b200 import api
    from paper_2602_08043_b200.fused import FusedAbftGemm, operand_faults
    m, k, n = 128, 256, 264
    A, B = port.trial_inputs(m, k, n, fmt, "normal:0,1", 29, bit)
    dt = torch.float64 if fmt == "fp64" else torch.float32
    npdt = np.float64 if fmt == "fp64" else np.float32
    udt = np.uint64 if fmt == "fp64" else np.uint32
    e_max = 4e-15 if fmt == "fp64" else 2e-6
    g = FusedAbftGemm(torch.from_numpy(B).to(dt).cuda(), e_max=e_max)
    dA = torch.from_numpy(A).to(dt).cuda()
    rng = np.random.default_rng(bit)
    Af, Bf = A.astype(npdt), B.astype(npdt)

    def flip(x, bitpos):
        return (np.array([x], dtype=npdt).view(udt) ^ udt(1 << bitpos)).view(npdt)[0]
    if target == "A":
        ks = rng.integers(0, k, m)
        for i, kk in enumerate(ks):
            Af[i, kk] = flip(Af[i, kk], bit)
        rec = torch.zeros(m * 24, dtype=torch.uint8, device="cuda")
        f = {"target": "A", "col": torch.from_numpy(ks.astype(np.int32)).cuda(),
             "bit": torch.full((m,), bit, dtype=torch.int32, device="cuda"),
             "dir": torch.zeros(m, dtype=torch.int32, device="cuda"), "records": rec}
    else:
        pos = [(int(rng.integers(0, k)), int(rng.integers(0, n))) for _ in range(3)]
        for (kk, j) in pos:
            Bf[kk, j] = flip(Bf[kk, j], bit)
        f = {"target": "B", "operand": operand_faults([(kk, j, bit, 0) for (kk, j) in pos])}
    counts = torch.zeros(6, dtype=torch.int64, device="cuda")
    r = g(dA, faults=f, checksums=True, counts=counts)
    torch.cuda.synchronize()
    Cf = r.C.double().cpu().numpy()
    e = api.encode_and_multiply(Af.astype(np.float64), Bf.astype(np.float64), "online", fmt, engine="tensor")
    assert same(Cf, e.c)  # the same kernel on the flipped operand
    o = port.encode_and_multiply(A, B, fmt, "online", accum=BLK)  # clean checksums
    assert same(r.row_check1.cpu().numpy(), o.row_check1)
    T_ref, _ = port.vabft_thresholds(A, B, e_max, fmt=fmt)
    assert same(r.T.cpu().numpy(), T_ref)
    v = port.verify(Cf, o.row_check1, o.row_check2, T_ref, fmt, "online", accum=BLK)
    assert np.array_equal(v["detected"], r.detected.cpu().numpy().astype(bool))
    assert np.array_equal(v["location"], r.location.cpu().numpy())
    assert int(counts[1].item()) == int(v["detected"].sum()) and v["detected"].any()


@pytest.mark.parametrize("fmt", ["fp32", "fp64"])
def test_wide_bside_row_sums_guard_and_fallback(torch_cuda, port, fmt):
    """B-side row statistics of a wide-format weight: rows whose order-free
    warp sum is exact under the guard, rows with tiny elements that take the
    sequential (batched-load) loops, a zero row and a row with a lone
    subnormal-scale element: thresholds and checksums bit-exact vs the oracle."""
    torch = torch_cuda
    from paper_2602_08043_b200.fused import FusedAbftGemm
    rng = np.random.default_rng(11)
    m, k, n = 64, 96, 1096  # ragged last 128-column block
    dt = np.float32 if fmt == "fp32" else np.float64
    B = rng.standard_normal((k, n)).astype(dt)
    B[3, ::7] *= dt(1e-12)
    B[5] = 0.0
    B[9] = 0.0
    B[9, 17] = dt(3e-30)
    B[11] = (rng.standard_normal(n) * 1e6).astype(dt)
    B[11, 1] = dt(1e-20)
    A = rng.standard_normal((m, k)).astype(dt)
    A64, B64 = A.astype(np.float64), B.astype(np.float64)
    e_max = 1e-5
    g = FusedAbftGemm(torch.from_numpy(B).cuda(), mode="online", e_max=e_max)
    r = g(torch.from_numpy(A).cuda(), checksums=True)
    torch.cuda.synchronize()
    T_ref, _ = port.vabft_thresholds(A64, B64, e_max, fmt=fmt)
    assert same(r.T.cpu().numpy(), T_ref)
    o = port.encode_and_multiply(A64, B64, fmt, "online", accum=BLK)
    assert same(r.row_check1.cpu().numpy(), o.row_check1) and same(r.row_check2.cpu().numpy(), o.row_check2)
    assert int(r.detected.sum().item()) == 0
