"""Operand faults and in-kernel correction against the
oracle.

A fault in the A / B operand as the tensor cores see it (the clean checksums
and statistics come from the unflipped operands) must give exactly the
verdicts the reference's verify() gives for C = A' B with the clean
encoding: the device accumulator of the flipped product (same tcgen05
kernel order) checked by the port against the clean row checksums, with the
FP32 NativeBlocked(128) checksum precision. Correction must reproduce
correct() (detect.cpp:57-64): C[i][j] = quantize(C[i][j] - diff1)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


def same(a, b):
    """bit-identical, NaN == NaN (payloads of NaN differences are not specified)"""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and np.array_equal(a[~na].view(np.uint64), b[~nb].view(np.uint64))


def bf16_bits(x):
    return (np.asarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def from_bits(b):
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("mode", ["online", "offline"])
@pytest.mark.parametrize("bit", [4, 10, 14])
def test_a_operand_faults_match_oracle(torch_cuda, port, mode, bit):
    torch = torch_cuda
    from paper_2602_08043_b200 import api
    from paper_2602_08043_b200.fused import FusedAbftGemm
    m, k, n = 128, 320, 512
    A, B = port.trial_inputs(m, k, n, "bf16", "normal:1e-6,1", 41, bit)
    rng = np.random.default_rng(bit)
    kk = rng.integers(0, k, m)
    kk[::7] = -1  # rows without a fault
    dA = torch.from_numpy(A).to(torch.bfloat16).cuda()
    dB = torch.from_numpy(B).to(torch.bfloat16).cuda()
    g = FusedAbftGemm(dB, mode=mode)
    rec = torch.zeros(m * 24, dtype=torch.uint8, device="cuda")
    f = {"target": "A", "col": torch.from_numpy(kk.astype(np.int32)).cuda(),
         "bit": torch.full((m,), bit, dtype=torch.int32, device="cuda"),
         "dir": torch.full((m,), 1, dtype=torch.int32, device="cuda"), "records": rec}
    r = g(dA, faults=f, checksums=True)
    torch.cuda.synchronize()
    applied = rec.view(m, 24)[:, 16:20].contiguous().view(torch.int32).view(m).cpu().numpy() != 0
    # the flipped operand on the host
    bits = bf16_bits(A)
    for i in range(m):
        if kk[i] >= 0 and not (bits[i, kk[i]] >> bit) & 1:
            bits[i, kk[i]] ^= np.uint16(1 << bit)
            assert applied[i]
        else:
            assert not applied[i]
    A2 = from_bits(bits)
    clean = api.encode_and_multiply(A, B, mode, "bf16", engine="tensor")
    dirty = api.encode_and_multiply(A2, B, "online", "bf16", engine="tensor")  # C and the accumulator
    assert same(r.row_check1.cpu().numpy(), clean.row_check1)  # checksums from the clean A
    src = dirty.c_accum if mode == "online" else dirty.c
    assert np.array_equal(r.C.cpu().to(torch.float32).numpy().astype(np.float64), dirty.c)
    v = port.verify(src, clean.row_check1, clean.row_check2, r.T.cpu().numpy(), "fp32", "offline", accum=(2, 128))
    assert same(r.diff1.cpu().numpy(), v["diff1"])
    assert np.array_equal(r.detected.cpu().numpy().astype(bool), v["detected"])
    assert np.array_equal(r.location.cpu().numpy(), v["location"])
    assert not r.detected.cpu().numpy().astype(bool)[~applied].any()  # clean rows: no false positive
    if bit == 14:  # an exponent bit of a BF16 operand: caught in every applied row
        assert r.detected.cpu().numpy().astype(bool)[applied].all()
    g.close()


@pytest.mark.parametrize("mode", ["online", "offline"])
def test_b_operand_faults_match_oracle(torch_cuda, port, mode):
    torch = torch_cuda
    from paper_2602_08043_b200 import api
    from paper_2602_08043_b200.fused import FusedAbftGemm, operand_faults
    m, k, n = 256, 192, 640
    A, B = port.trial_inputs(m, k, n, "bf16", "normal:1e-6,1", 43, 0)
    faults = [(5, 17, 13, 0), (100, 300, 9, 0), (191, 639, 14, 0)]  # (k, j, bit, Flip)
    dA = torch.from_numpy(A).to(torch.bfloat16).cuda()
    dB = torch.from_numpy(B).to(torch.bfloat16).cuda()
    g = FusedAbftGemm(dB, mode=mode)
    rec = torch.zeros(len(faults) * 24, dtype=torch.uint8, device="cuda")
    r = g(dA, faults={"target": "B", "operand": operand_faults(faults), "records": rec}, checksums=True)
    torch.cuda.synchronize()
    assert (rec.view(len(faults), 24)[:, 16:20].contiguous().view(torch.int32).cpu().numpy() == 1).all()
    bits = bf16_bits(B)
    for (kk, j, bit, _) in faults:
        bits[kk, j] ^= np.uint16(1 << bit)
    B2 = from_bits(bits)
    clean = api.encode_and_multiply(A, B, mode, "bf16", engine="tensor")
    dirty = api.encode_and_multiply(A, B2, "online", "bf16", engine="tensor")
    src = dirty.c_accum if mode == "online" else dirty.c
    v = port.verify(src, clean.row_check1, clean.row_check2, r.T.cpu().numpy(), "fp32", "offline", accum=(2, 128))
    assert same(r.diff1.cpu().numpy(), v["diff1"]) and same(r.diff2.cpu().numpy(), v["diff2"])
    assert np.array_equal(r.detected.cpu().numpy().astype(bool), v["detected"])
    assert np.array_equal(r.location.cpu().numpy(), v["location"])
    g.close()


def test_in_kernel_correction_matches_correct(torch_cuda, port):
    torch = torch_cuda
    from paper_2602_08043_b200 import _capi
    from paper_2602_08043_b200.fused import FusedAbftGemm
    m, k, n = 256, 512, 384
    A, B = port.trial_inputs(m, k, n, "bf16", "normal:1e-6,1", 47, 0)
    dA = torch.from_numpy(A).to(torch.bfloat16).cuda()
    dB = torch.from_numpy(B).to(torch.bfloat16).cuda()
    g = FusedAbftGemm(dB, mode="offline")
    clean = g(dA).C.clone()
    rng = np.random.default_rng(3)
    cols = rng.integers(0, n, m)
    f = {"col": torch.from_numpy(cols.astype(np.int32)).cuda(),
         "bit": torch.full((m,), 13, dtype=torch.int32, device="cuda"),
         "dir": torch.full((m,), 0, dtype=torch.int32, device="cuda")}  # Flip: always applied
    counts = torch.zeros(_capi.NUM_COUNTS, dtype=torch.int64, device="cuda")
    faulty = g(dA, faults=f).C.clone()
    r = g(dA, faults=f, correct=True, counts=counts)
    torch.cuda.synchronize()
    C = r.C.cpu().to(torch.float32).numpy().astype(np.float64)
    Cf = faulty.cpu().to(torch.float32).numpy().astype(np.float64)
    d1 = r.diff1.cpu().numpy()
    loc = r.location.cpu().numpy()
    res = r.residual.cpu().numpy()
    fixed = 0
    for i in range(m):
        exp_row = Cf[i].copy()
        if loc[i] >= 0 and res[i] < 0.4:
            exp_row[loc[i]] = port.quantize(Cf[i, loc[i]] - d1[i], "bf16")  # correct(), detect.cpp:57-64
            fixed += 1
        assert np.array_equal(C[i], exp_row)
    assert counts[_capi.COUNT_CORRECTED].item() == fixed and fixed > 0.9 * m
    # a bit-13 flip of a BF16 output is a clean single error: correction restores
    # it up to the clean row's rounding noise carried in diff1
    assert (C == clean.cpu().to(torch.float32).numpy()).mean() > 0.99
    g.close()
