"""GPU fault-injection campaigns (faults.cpp:104-216) against the oracle.

Per-trial parity: the fused kernel's verdict for every injected row equals
the reference's verify() applied to the same device accumulator / output with
the same bit flip (FP32 NativeBlocked(128) checksum precision) — bit-exact.
Campaign statistics: detection is ~100% for high exponent bits and the
location is recovered, FPR stays 0 for rows whose flip was not applicable."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


def _flip_bits(vals, cols, bit, fmt, direction, port):
    """Reference inject() at fixed positions (faults.cpp:104-168), one per row."""
    out = vals.copy()
    applied = np.zeros(len(cols), dtype=bool)
    for i, j in enumerate(cols):
        X, rec = port.inject(out[i:i + 1], fmt, bit, direction=direction, pos=(0, int(j)), src_fp32=(fmt == "fp32"))
        out[i:i + 1] = X
        applied[i] = rec["applied"]
    return out, applied


@pytest.mark.parametrize("mode", ["online", "offline"])
@pytest.mark.parametrize("bit", [3, 12, 20, 29])
def test_fused_injection_matches_oracle_per_trial(torch_cuda, port, mode, bit):
    torch = torch_cuda
    from paper_2602_08043_b200 import api
    from paper_2602_08043_b200.fused import FusedAbftGemm
    m, k, n = 128, 256, 384
    if mode == "offline" and bit >= 16:
        bit = bit % 16
    A, B = port.trial_inputs(m, k, n, "bf16", "normal:1e-6,1", 31, bit)
    rng = np.random.default_rng(bit)
    cols = rng.integers(0, n, m)
    dA = torch.from_numpy(A).to(torch.bfloat16).cuda()
    dB = torch.from_numpy(B).to(torch.bfloat16).cuda()
    g = FusedAbftGemm(dB, mode=mode)
    rec = torch.empty(m * 24, dtype=torch.uint8, device="cuda")
    f = {"col": torch.from_numpy(cols.astype(np.int32)).cuda(),
         "bit": torch.full((m,), bit, dtype=torch.int32, device="cuda"),
         "dir": torch.full((m,), 1, dtype=torch.int32, device="cuda"), "records": rec}
    r = g(dA, faults=f, checksums=True)
    torch.cuda.synchronize()
    det = r.detected.cpu().numpy().astype(bool)
    loc = r.location.cpu().numpy()
    T = r.T.cpu().numpy()
    rc1, rc2 = r.row_check1.cpu().numpy(), r.row_check2.cpu().numpy()
    applied_dev = rec.view(m, 24)[:, 16:20].contiguous().view(torch.int32).view(m).cpu().numpy() != 0
    # the same accumulator through the parity API (same kernel, same MMA order)
    e = api.encode_and_multiply(A, B, mode, "bf16", engine="tensor")
    assert np.array_equal(rc1.view(np.uint64), e.row_check1.view(np.uint64))
    src = e.c_accum if mode == "online" else e.c
    flipped, applied = _flip_bits(src, cols, bit, "fp32" if mode == "online" else "bf16", 1, port)
    assert np.array_equal(applied, applied_dev)
    v = port.verify(flipped, rc1, rc2, T, "fp32", "offline", accum=(2, 128))
    assert np.array_equal(v["detected"], det)
    assert np.array_equal(v["location"], loc)
    # rows whose flip was not applicable are clean: no false positives there
    assert not det[~applied].any()


def test_campaign_rates(torch_cuda):
    from paper_2602_08043_b200.campaign import DeviceCampaign
    c = DeviceCampaign(256, 1024, 256, dist="normal:1e-6,1", mode="online", seed=5)
    hi = c.run(29, 512, reduce=False)   # FP32 exponent bit 6: |x| in [2^-62, 2) -> x 2^64
    lo = c.run(0, 512, reduce=False)    # FP32 mantissa LSB: below every threshold
    mid = c.run(24, 512, reduce=False)  # exponent LSB: doubles/halves the value
    c.close()
    assert hi.applicable > 200 and hi.detection_rate() == 1.0 and hi.localization_accuracy() > 0.99
    assert lo.applicable > 100 and lo.detection_rate() == 0.0
    assert mid.detection_rate() > 0.99 and mid.localization_accuracy() > 0.99


@pytest.mark.parametrize("mode", ["online", "offline"])
@pytest.mark.parametrize("shape", [(512, 1024, 1024), (384, 512, 768), (4096, 512, 4096), (2560, 256, 4000)])
def test_cta_pair_and_one_cta_kernels_agree(torch_cuda, mode, shape):
    """The CTA-pair (cta_group::2) and one-CTA fused kernels run the same MMA
    order per output, statistics and verification: C, thresholds, differences
    and verdicts are bit-identical. The last two shapes leave the pair grid's
    last wave under half full (256 and 160 pair tiles over 74 pairs), so their
    last tiles run as 128-column halves (the second with a ragged N edge)."""
    torch = torch_cuda
    from paper_2602_08043_b200.fused import FusedAbftGemm
    m, k, n = shape
    torch.manual_seed(3)
    A = torch.randn(m, k, device="cuda").bfloat16()
    B = torch.randn(k, n, device="cuda").bfloat16()
    g = FusedAbftGemm(B, mode=mode)
    out = {}
    for cm in (0, 1):
        g.opts.cta_mode = cm
        r = g(A, out=torch.empty(m, n, device="cuda", dtype=torch.bfloat16))
        torch.cuda.synchronize()
        out[cm] = (r.C.clone(), r.T.clone(), r.diff1.clone(), r.detected.clone())
    assert g.uses_cta_pairs(m)
    c0, c1 = out[0], out[1]
    assert torch.equal(c0[0].view(torch.int16), c1[0].view(torch.int16))
    assert torch.equal(c0[1], c1[1]) and torch.equal(c0[2], c1[2]) and torch.equal(c0[3], c1[3])


@pytest.mark.parametrize("cta_mode", [0, 1])
def test_statistics_across_magnitudes_bit_exact(torch_cuda, port, cta_mode):
    """Row statistics inside the GEMM (integer images of the elements, the
    exactness guard and its sequential fallback) across row magnitudes from
    BF16 subnormals to 2^60, zero rows and mixed-scale rows: thresholds
    bit-identical to the oracle's vabft_thresholds."""
    torch = torch_cuda
    from paper_2602_08043_b200.fused import FusedAbftGemm
    m, k, n = 256, 512, 512
    rng = np.random.default_rng(11)
    A = rng.standard_normal((m, k))
    scales = [2.0**-130, 2.0**-100, 2.0**-75, 2.0**-70, 1e-30, 1e-6, 1.0, 2.0**20, 2.0**60]
    for i in range(m):
        A[i] *= scales[i % len(scales)]
    A[5] = 0.0                                   # zero row
    A[6, ::2] *= 2.0**-40                        # mixed scales inside a row
    A[7, :64] *= 2.0**-60                        # one tiny stage
    A = np.array([port.quantize(x, "bf16") for x in A.ravel()]).reshape(m, k)
    B = np.array([port.quantize(x, "bf16") for x in rng.standard_normal((k, n)).ravel()]).reshape(k, n)
    g = FusedAbftGemm(torch.from_numpy(B).to(torch.bfloat16).cuda(), e_max=1e-5)
    g.opts.cta_mode = cta_mode
    r = g(torch.from_numpy(A).to(torch.bfloat16).cuda())
    torch.cuda.synchronize()
    T_ref, _ = port.vabft_thresholds(A, B, 1e-5, fmt="bf16")
    T = r.T.cpu().numpy()
    assert np.array_equal(T.view(np.uint64), T_ref.view(np.uint64)), np.where(T != T_ref)[0][:8]
