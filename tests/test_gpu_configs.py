"""Oracle parity of the default fused kernel at the BASELINE.json configs.

The production launch (CTA pairs, cta_group::2 on 256 x 256 tiles, the
under-filled last wave as 128-column half tiles, statistics warps, streamed
verification inside the GEMM) runs the full shapes of

  C1  FP32 1024^3 (3xTF32 on tcgen05) with single bit flips, bits 0..31
  C2  BF16 4096^3, online (FP32 accumulator) and offline (BF16 output)
  C4  LLaMA-7B layer GEMMs, tokens M = 8192: (K, N) = (4096, 11008), (11008, 4096)
  C5  ViT-B/16 (M = 32 * 197 = 6304, ragged) and GPT-2 (M = 1024) layer shapes
      (+ FP16 / FP64 at 2048^3 from the C3 sweep)

and is compared with the reference compiled from its own sources
(oracle/_ref; the C restatement where it is not built) on a row sample S.
Rows of a GEMM are independent sub-problems of every reference function on
the path, so the reference runs on A[S] with the full B:

  T          = vabft_thresholds(A[S], B)             (threshold_vabft.cpp:54-61)   bit-exact
  row checks = A[S] (B r) in the fused path's FP32 NativeBlocked(128) checksum
               precision, composed from the reference's row_sums
               (checksum.cpp:103-187)                                              bit-exact
  verdicts   = verify(device accumulator / output [S], row checks, T)
               (detect.cpp:9-55): diff1, diff2, residual, detected, location   bit-exact
  C          = within the FP32-accumulate bound of test_precision.cpp:181-206
               against the exact product; C == RNE(accumulator) bit for bit.

Planted faults (one per faulted row, accumulator bits online, output bits
offline) land in sampled rows, so their verdicts and located columns are
compared too; every other row of the full matrix is clean and must not be
flagged (FPR = 0 over all M rows).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BITS_ONLINE = [0, 7, 12, 14, 15, 16, 18, 20, 22, 23, 24, 26, 28, 29, 30, 31]
BITS_OFFLINE = [0, 3, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15]


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available()
    import oracle
    return torch, oracle.best()


def _same(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and np.array_equal(a[~na].view(np.uint64), b[~nb].view(np.uint64))


def _sample_rows(m, rng, count=48):
    """Random rows + the first rows + the last 256-row (pair) block, which
    holds the ragged M tail and, at split shapes, rows of the half tiles."""
    if m <= 1024:
        return np.arange(m)  # C1 and the GPT-2 shapes: every row
    rows = set(rng.choice(m, size=min(count, m), replace=False).tolist())
    rows.update(range(min(4, m)))
    last = max(0, (m - 1) // 256 * 256)
    rows.update(rng.choice(np.arange(last, m), size=min(12, m - last), replace=False).tolist())
    rows.add(m - 1)
    return np.array(sorted(rows))


def _inputs(torch, m, k, n, dt, seed, weights="normal"):
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.randn(m, k, device="cuda", generator=g, dtype=torch.float32)
    if weights == "linear":  # nn.Linear default init
        B = (torch.rand(k, n, device="cuda", generator=g) * 2 - 1) / k ** 0.5
    else:
        B = torch.randn(k, n, device="cuda", generator=g, dtype=torch.float32)
    if dt == torch.float64:
        return A.double(), B.double()
    return A.to(dt), B.to(dt)


def _run_config(env, m, k, n, fmt, mode, seed, weights="normal", faulted_fraction=0.5, tf32_passes=3):
    torch, O = env
    from paper_2602_08043_b200.fused import FusedAbftGemm
    dt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32, "fp64": torch.float64}[fmt]
    dA, dB = _inputs(torch, m, k, n, dt, seed, weights)
    rng = np.random.default_rng(seed)
    S = _sample_rows(m, rng)
    g = FusedAbftGemm(dB, mode=mode, tf32_passes=tf32_passes)
    wide = fmt in ("fp32", "fp64")
    if not wide:
        assert g.uses_cta_pairs(m), "the default launch must be the CTA-pair kernel"
    # planted faults in a subset of the sampled rows
    fr = S[rng.random(len(S)) < faulted_fraction]
    bits = BITS_ONLINE if (mode == "online" or fmt == "fp32") else BITS_OFFLINE
    if fmt == "fp64":
        bits = [0, 20, 40, 45, 50, 52, 55, 58, 60, 62]
    col = torch.full((m,), -1, dtype=torch.int32)
    bit = torch.zeros(m, dtype=torch.int32)
    fcols = rng.integers(0, n, len(fr))
    fbits = rng.choice(bits, len(fr))
    col[torch.from_numpy(fr)] = torch.from_numpy(fcols.astype(np.int32))
    bit[torch.from_numpy(fr)] = torch.from_numpy(fbits.astype(np.int32))
    faults = {"col": col.cuda(), "bit": bit.cuda(), "dir": torch.zeros(m, dtype=torch.int32, device="cuda")}
    counts = torch.zeros(6, dtype=torch.int64, device="cuda")
    acc = None if wide else torch.empty(m, n, dtype=torch.float32, device="cuda")
    r = g(dA, counts=counts, checksums=True, faults=faults, accum_out=acc)
    torch.cuda.synchronize()
    e_max = g.opts.e_max
    Sd = torch.from_numpy(S).cuda()
    A_s = dA[Sd].double().cpu().numpy()
    B_h = dB.double().cpu().numpy()
    dev = {k_: getattr(r, k_)[Sd].cpu().numpy() for k_ in ("T", "diff1", "diff2", "residual", "location",
                                                           "row_check1", "row_check2")}
    det = r.detected.cpu().numpy().astype(bool)
    # --- oracle on the row sample
    T_ref, _ = O.vabft_thresholds(A_s, B_h, e_max, fmt=fmt)
    assert _same(dev["T"], T_ref), ("thresholds", S[np.flatnonzero(dev["T"] != T_ref)][:8])
    rc1, rc2 = O.blocked_row_checksums(A_s, B_h, fmt, mode)
    assert _same(dev["row_check1"], rc1) and _same(dev["row_check2"], rc2), "row checksums"
    if wide:
        src = r.C[Sd].double().cpu().numpy()
        v = O.verify(src, rc1, rc2, T_ref, fmt, "online", accum=(2, 128))
    else:
        src = (acc[Sd] if mode == "online" else r.C[Sd]).double().cpu().numpy()
        v = O.verify(src, rc1, rc2, T_ref, "fp32", "offline", accum=(2, 128))
    for key in ("diff1", "diff2", "residual"):
        assert _same(dev[key], v[key]), key
    assert np.array_equal(det[S], v["detected"]), ("detected", S[det[S] != v["detected"]][:8])
    assert np.array_equal(dev["location"], v["location"]), "location"
    # --- FPR over the full matrix: only planted rows may be flagged
    clean = np.ones(m, dtype=bool)
    clean[fr] = False
    assert not det[clean].any(), ("false positives", np.flatnonzero(det & clean)[:8])
    assert int(counts[0].item()) == m and int(counts[1].item()) == int(det.sum())
    # --- C: FP32-accumulate bound against the exact product (unfaulted elements)
    exact = A_s @ B_h
    bound = (k + 1) * 2.0**-24 * (np.abs(A_s) @ np.abs(B_h))
    got = src if (wide or mode == "online") else acc[Sd].double().cpu().numpy()
    mask = np.ones_like(got, dtype=bool)
    for i_s, row in enumerate(S):
        if col[row] >= 0:
            mask[i_s, int(col[row])] = False
    assert np.all(np.abs(got - exact)[mask] <= bound[mask])
    if not wide:  # C is the saturating RNE quantization (precision.cpp:129-159) of the post-injection accumulator
        fmax = 65504.0 if fmt == "fp16" else float(torch.finfo(torch.bfloat16).max)
        q = acc.clamp(-fmax, fmax).to(dt)
        if mode == "offline":  # output-bit faults land after quantization
            q[torch.from_numpy(fr).cuda(), torch.from_numpy(fcols).cuda()] = r.C[torch.from_numpy(fr).cuda(),
                                                                                  torch.from_numpy(fcols).cuda()]
        nan = torch.isnan(q)
        assert torch.equal(torch.isnan(r.C), nan)
        assert torch.equal(r.C.view(torch.int16)[~nan], q.view(torch.int16)[~nan])
    located = v["location"][np.isin(S, fr)]
    want = fcols[np.searchsorted(fr, S[np.isin(S, fr)])]
    g.close()
    return {"rows": len(S), "faulted": len(fr), "detected": int(v["detected"][np.isin(S, fr)].sum()),
            "located": int((located == want).sum())}


@pytest.mark.parametrize("mode", ["online", "offline"])
def test_c2_bf16_4096_cubed(env, mode):
    out = _run_config(env, 4096, 4096, 4096, "bf16", mode, seed=2)
    assert out["detected"] > 0 and out["located"] > 0


@pytest.mark.parametrize("k,n", [(4096, 11008), (11008, 4096)])
def test_c4_llama_layer_shapes(env, k, n):
    out = _run_config(env, 8192, k, n, "bf16", "online", seed=k + n, weights="linear")
    assert out["detected"] > 0


@pytest.mark.parametrize("m,k,n", [(6304, 768, 3072), (6304, 3072, 768), (6304, 768, 2304), (1024, 768, 2304),
                                   (1024, 3072, 768)])
def test_c5_vit_gpt2_shapes(env, m, k, n):
    _run_config(env, m, k, n, "bf16", "online", seed=m + k + n)


def test_c1_fp32_1024_cubed_bit_flips(env):
    """C1: FP32 1024^3 N(0,1), 3xTF32 on tcgen05, single bit flips over bits
    0..31 in half of all rows (every row is sampled)."""
    out = _run_config(env, 1024, 1024, 1024, "fp32", "online", seed=1, faulted_fraction=0.5)
    assert out["detected"] > 0 and out["located"] > 0


@pytest.mark.parametrize("fmt", ["fp16", "fp64"])
def test_c3_other_formats_2048(env, fmt):
    _run_config(env, 2048, 2048, 2048, fmt, "online", seed=5)


@pytest.mark.parametrize("mode", ["online", "offline"])
def test_pair_half_tiles_match_one_cta_at_k4096(env, mode):
    """4096^3 is 256 pair tiles = 3 waves of 74 + 34: the last 34 run as 68
    half tiles, whose statistics warps take every other 128-k block of their
    tile (K = 4096: 32 blocks over 16 N tiles, so the half-tile branch runs).
    Thresholds, differences, verdicts and C equal the one-CTA kernel's."""
    torch, _ = env
    from paper_2602_08043_b200.fused import FusedAbftGemm
    dA, dB = _inputs(torch, 4096, 4096, 4096, torch.bfloat16, 9)
    g = FusedAbftGemm(dB, mode=mode)
    out = {}
    for cm in (0, 1):
        g.opts.cta_mode = cm
        r = g(dA, out=torch.empty(4096, 4096, device="cuda", dtype=torch.bfloat16), checksums=True)
        torch.cuda.synchronize()
        out[cm] = [x.clone() for x in (r.C.view(torch.int16), r.T, r.diff1, r.diff2, r.detected, r.row_check1)]
    for a, b in zip(out[0], out[1]):
        assert torch.equal(a, b)
    g.close()


def test_guard_failing_rows_at_c2_size(env):
    """Rows whose A statistics fail the in-GEMM exactness guard (entries near
    1e-10 next to O(1) ones at K = 4096) take the warp-cooperative Neumaier
    rerun inside the streamed verification: thresholds stay bit-exact against
    the reference and the rerun count is reported in counts[4]."""
    torch, O = env
    from paper_2602_08043_b200.fused import FusedAbftGemm
    m = k = n = 4096
    dA, dB = _inputs(torch, m, k, n, torch.bfloat16, 21)
    rows = torch.arange(0, m, 61, device="cuda")  # 68 rows
    tiny = (torch.rand(len(rows), k, device="cuda") < 0.5)
    dA[rows] = torch.where(tiny, dA[rows].float() * 1e-10, dA[rows].float()).bfloat16()
    g = FusedAbftGemm(dB)
    counts = torch.zeros(6, dtype=torch.int64, device="cuda")
    r = g(dA, counts=counts)
    torch.cuda.synchronize()
    assert int(counts[4].item()) >= len(rows) // 2, counts.tolist()
    S = torch.cat([rows[:24], torch.arange(1, 40, device="cuda")]).unique()
    T_ref, _ = O.vabft_thresholds(dA[S].double().cpu().numpy(), dB.double().cpu().numpy(), g.opts.e_max, fmt="bf16")
    assert _same(r.T[S].cpu().numpy(), T_ref)
    assert int(counts[1].item()) == 0
    g.close()


@pytest.mark.parametrize("fmt", ["bf16", "fp16", "fp32", "fp64"])
@pytest.mark.parametrize("shape", [(1024, 1000), (300, 777)])
def test_bside_pass_mixed_scales_bit_exact(env, fmt, shape):
    """The per-weight B-side pass (bside.cu) on weights whose rows mix
    magnitudes far apart (rows outside the exactness guard go through the
    warp Neumaier rerun) and odd / ragged N: B summary and thresholds
    bit-exact against the reference's precompute_b_stats / BStatsSummary."""
    torch, O = env
    from paper_2602_08043_b200 import api
    k, n = shape
    rng = np.random.default_rng(k + n)
    B = rng.standard_normal((k, n))
    B[::7] *= np.where(rng.random((len(B[::7]), n)) < 0.3, 1e-9, 1.0)
    B[3::11] *= 1e-25 if fmt != "fp16" else 1e-4
    A = rng.standard_normal((64, k))
    B = np.array([O.quantize(x, fmt) for x in B.ravel()]).reshape(B.shape)
    A = np.array([O.quantize(x, fmt) for x in A.ravel()]).reshape(A.shape)
    T, summ = api.vabft_thresholds(A, B, api.VabftParams(1e-3, 2.5), fmt, return_summary=True)
    T_ref, s_ref = O.vabft_thresholds(A, B, 1e-3, fmt=fmt)
    assert _same(summ, s_ref)
    assert _same(T, T_ref)


@pytest.mark.parametrize("k", [700, 4096])
def test_bside_summary_chain_adversarial(env, k):
    """BStatsSummary's three sequential FP64 sums (threshold_vabft.cpp:19-24)
    folded from the published row groups through the summary warps' cp.async
    ring (bside.cu bs_summary), on terms that stress a sequential sum: leading
    zero rows, tiny rows (1e-300), runs of ties against the running sum
    (1 + 2^-52 while the sum is in [2, 4)), binade crossings, huge jumps and
    random magnitudes, with K not a multiple of the 256-row batch. FP64 rows
    [v, v] give mean v and var_bound 0; other rows [v, w] give var_bound > 0."""
    torch, O = env
    from paper_2602_08043_b200 import api
    rng = np.random.default_rng(k)
    v = np.empty(k)
    w = np.empty(k)
    i = 0
    for blk in range(k):
        kind = (blk * 7919) % 11
        if blk < 5:
            x = 0.0
        elif blk < 9:
            x = 1e-300 * (blk - 4)
        elif kind < 4:
            x = 1.0 + 2.0 ** -52
        elif kind == 4:
            x = 2.0 ** int(rng.integers(-40, 40))
        elif kind == 5:
            x = float(rng.standard_normal()) * 1e6
        else:
            x = float(rng.standard_normal())
        v[i] = x
        w[i] = x if kind % 2 == 0 else x + float(rng.standard_normal()) * 2.0 ** -20
        i += 1
    B = np.stack([v, w], axis=1)
    A = rng.standard_normal((64, k))
    T, summ = api.vabft_thresholds(A, B, api.VabftParams(1e-3, 2.5), "fp64", return_summary=True)
    T_ref, s_ref = O.vabft_thresholds(A, B, 1e-3, fmt="fp64")
    assert _same(summ, s_ref), (summ, s_ref)
    assert _same(T, T_ref)


def test_nsplit_slices_match_oracle_on_slices(env):
    """SURVEY §8(e) N-sharding: two column slices of one C4-shaped GEMM
    (8192 x 4096 x 11008 split by shard_columns), each a ColumnShardedGemm
    verifying its slice as an independent ABFT unit. Per slice, thresholds,
    checksums and verdicts equal the reference on (A[S], B[:, n0:n1]); planted
    faults are located at their GLOBAL column; C slices reassemble the full
    product bit for bit (one-rank run of the same two slices)."""
    torch, O = env
    from paper_2602_08043_b200.sharding import ColumnShardedGemm, shard_columns
    m, k, n = 8192, 4096, 11008
    dA, dB = _inputs(torch, m, k, n, torch.bfloat16, 44, weights="linear")
    rng = np.random.default_rng(44)
    S = _sample_rows(m, rng, count=24)
    A_s = dA[torch.from_numpy(S).cuda()].double().cpu().numpy()
    B_h = dB.double().cpu().numpy()
    C_full = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    for n0, n1 in shard_columns(n, 2):
        sg = ColumnShardedGemm(dB[:, n0:n1].contiguous(), n0, n)
        col = torch.full((m,), -1, dtype=torch.int32, device="cuda")
        bit = torch.zeros(m, dtype=torch.int32, device="cuda")
        fr = S[::3]
        fc = rng.integers(0, n1 - n0, len(fr))
        col[torch.from_numpy(fr).cuda()] = torch.from_numpy(fc.astype(np.int32)).cuda()
        bit[torch.from_numpy(fr).cuda()] = 26  # flip exponent bit 3: x 2^+-8
        out = torch.empty(m, n1 - n0, dtype=torch.bfloat16, device="cuda")
        acc = torch.empty(m, n1 - n0, dtype=torch.float32, device="cuda")
        r = sg(dA, out=out, checksums=True, accum_out=acc,
               faults={"col": col, "bit": bit, "dir": torch.zeros(m, dtype=torch.int32, device="cuda")})
        torch.cuda.synchronize()
        Sd = torch.from_numpy(S).cuda()
        Bs = B_h[:, n0:n1]
        T_ref, _ = O.vabft_thresholds(A_s, Bs, sg.g.opts.e_max, fmt="bf16")
        rc1, rc2 = O.blocked_row_checksums(A_s, Bs, "bf16", "online")
        assert _same(r.T[Sd].cpu().numpy(), T_ref)
        assert _same(r.row_check1[Sd].cpu().numpy(), rc1) and _same(r.row_check2[Sd].cpu().numpy(), rc2)
        v = O.verify(acc[Sd].double().cpu().numpy(), rc1, rc2, T_ref, "fp32", "offline", accum=(2, 128))
        assert np.array_equal(r.detected[Sd].cpu().numpy().astype(bool), v["detected"])
        assert np.array_equal(r.location[Sd].cpu().numpy(), v["location"])
        gl = sg.global_location(r).cpu().numpy()
        loc_fr = r.location.cpu().numpy()[fr]
        ok = loc_fr >= 0  # located unless |x| sits below the threshold
        assert ok.mean() > 0.7, (ok.sum(), len(fr))
        # the global column is the fault's (slice offset applied); a flip of a
        # small element (|D1| below the row-sum rounding noise of D2) can be
        # located elsewhere — by the reference too (device == oracle above)
        hit = gl[fr][ok] == (fc + n0)[ok]
        assert hit.any()
        assert np.array_equal(gl[fr][ok] - n0, loc_fr[ok])
        sg(dA, out=out)  # a clean run for the reassembly check below
        torch.cuda.synchronize()
        C_full[:, n0:n1] = out
        # clean rows stay clean
        det = r.detected.cpu().numpy().astype(bool)
        det[fr] = False
        assert not det.any()
        sg.close()
    # the slices reassemble the unsplit product (each C element is computed
    # independently of the other columns)
    ref = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    from paper_2602_08043_b200.fused import plain_gemm
    plain_gemm(dA, dB, out=ref)
    torch.cuda.synchronize()
    assert torch.equal(C_full.view(torch.int16), ref.view(torch.int16))


@pytest.mark.parametrize("n", [256, 1024])
def test_fp16_offline_normal_1_1_false_positives_are_the_references(env, n):
    """FP16 offline on N(1,1) operands flags clean rows — reference behaviour,
    not a kernel defect: offline row checksums A (B r2) are quantized to FP16
    and saturate at 65504 (checksum.cpp:129-134, precision.cpp:153-157), so
    D2 (and with it D1 for large rows) is wrong by construction. Per row, the
    fused kernel's verdicts equal the reference's verify on the same inputs
    (device output, reference thresholds and checksums), and the reference's
    own end-to-end pipeline (its emulated GEMM) flags rows too."""
    torch, O = env
    from paper_2602_08043_b200.fused import FusedAbftGemm
    A, B = O.trial_inputs(n, n, n, "fp16", "normal:1,1", 0, 0)
    g = FusedAbftGemm(torch.from_numpy(B).to(torch.float16).cuda(), mode="offline")
    counts = torch.zeros(6, dtype=torch.int64, device="cuda")
    r = g(torch.from_numpy(A).to(torch.float16).cuda(), counts=counts, checksums=True)
    torch.cuda.synchronize()
    e_max = g.opts.e_max
    T_ref, _ = O.vabft_thresholds(A, B, e_max, fmt="fp16")
    rc1, rc2 = O.blocked_row_checksums(A, B, "fp16", "offline")
    assert _same(r.T.cpu().numpy(), T_ref)
    assert _same(r.row_check1.cpu().numpy(), rc1) and _same(r.row_check2.cpu().numpy(), rc2)
    v = O.verify(r.C.double().cpu().numpy(), rc1, rc2, T_ref, "fp32", "offline", accum=(2, 128))
    det = r.detected.cpu().numpy().astype(bool)
    assert np.array_equal(det, v["detected"]) and np.array_equal(r.location.cpu().numpy(), v["location"])
    assert det.sum() > 0 and int(counts[1].item()) == det.sum()
    assert np.abs(rc2).max() == 65504.0  # the saturated checksums behind the flags
    e = O.encode_and_multiply(A, B, "fp16", "offline")  # the reference end to end
    T_full, _ = O.vabft_thresholds(A, B, e_max, fmt="fp16")
    vr = O.verify(e.c, e.row_check1, e.row_check2, T_full, "fp16", "offline")
    assert vr["detected"].sum() > 0
    g.close()


def test_bside_update_replayed_from_a_cuda_graph(env):
    """vabft_bside_update captured once in a CUDA graph and replayed with new
    weight values in the same buffer: the B-side pass keeps its launch epoch
    on the device, so every replay republishes its row groups and the
    thresholds stay bit-exact against the reference for each weight."""
    torch, O = env
    from paper_2602_08043_b200.fused import FusedAbftGemm
    m, k, n = 256, 1024, 768
    A, _ = _inputs(torch, m, k, n, torch.bfloat16, 61)
    Bbuf = torch.empty(k, n, device="cuda", dtype=torch.bfloat16)
    Bbuf.copy_(torch.randn(k, n, device="cuda"))
    g = FusedAbftGemm(Bbuf)
    g.update_weight(Bbuf)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        g.update_weight(Bbuf)
    for seed in (1, 2, 3):
        gen = torch.Generator(device="cuda").manual_seed(seed)
        Bbuf.copy_(torch.randn(k, n, device="cuda", generator=gen) * (seed + 1))
        gr.replay()
        r = g(A)
        torch.cuda.synchronize()
        T_ref, _ = O.vabft_thresholds(A.double().cpu().numpy(), Bbuf.double().cpu().numpy(), g.opts.e_max, fmt="bf16")
        assert _same(r.T.cpu().numpy(), T_ref), seed
    g.close()


@pytest.mark.parametrize("mode", ["online", "offline"])
def test_leading_dimensions_match_dense_calls(env, mode):
    """Row-strided operands (C-ABI v2 lda / ldc, vabft_bside_create_ld):
    A = a column window of a wider activation, B = a column slice of a wider
    weight, C written into the matching slice of a wider output — no copies;
    C, thresholds, checksums and verdicts equal the dense call's bit for bit
    (and the reference's on the slice, through the dense call's parity)."""
    torch, O = env
    from paper_2602_08043_b200.fused import FusedAbftGemm
    m, k, n, n0 = 1024, 768, 1536, 512
    Afull, Bfull = _inputs(torch, m, 2 * k, 2 * n, torch.bfloat16, 71)
    A = Afull[:, 128:128 + k]            # lda = 2K
    B = Bfull[:k, n0:n0 + n]             # ldb = 2N
    assert not A.is_contiguous() and not B.is_contiguous()
    g_s = FusedAbftGemm(B, mode=mode)
    assert g_s.ldb == 2 * n
    Cfull = torch.zeros(m, 2 * n, dtype=torch.bfloat16, device="cuda")
    r_s = g_s(A, out=Cfull[:, n0:n0 + n], checksums=True)
    torch.cuda.synchronize()
    got = [x.clone() for x in (r_s.T, r_s.diff1, r_s.detected, r_s.row_check1, r_s.row_check2)]
    g_d = FusedAbftGemm(B.contiguous(), mode=mode)
    r_d = g_d(A.contiguous(), checksums=True)
    torch.cuda.synchronize()
    assert torch.equal(Cfull[:, n0:n0 + n].view(torch.int16), r_d.C.view(torch.int16))
    assert torch.equal(Cfull[:, :n0], torch.zeros_like(Cfull[:, :n0]))  # nothing written outside the slice
    for a, b in zip(got, (r_d.T, r_d.diff1, r_d.detected, r_d.row_check1, r_d.row_check2)):
        assert torch.equal(a, b)
    g_s.close()
    g_d.close()


def test_guard_failing_tie_rows_bit_exact(env):
    """BF16 rows of O(1) and ~1e-10 entries whose exact sum lies EXACTLY on a
    rounding midpoint of doubles (about one such row in seven): a margin test
    cannot decide them, the integer exact sum inside the fused GEMM does
    (tail.cuh warp_exact_sum16: the reference's Neumaier compensation adds
    exactly for these rows, so fl(sum + comp) = fl(E), ties to even).
    Thresholds of the tie rows bit-exact against the reference's
    vabft_thresholds (stats.cpp:12-24, threshold_vabft.cpp:54-61)."""
    from fractions import Fraction

    torch, O = env
    from paper_2602_08043_b200.fused import FusedAbftGemm
    m, k, n = 512, 4096, 512
    dA, dB = _inputs(torch, m, k, n, torch.bfloat16, 33)
    rows = torch.arange(0, m, 4, device="cuda")  # 128 rows
    g = torch.Generator(device="cuda").manual_seed(34)
    tiny = torch.rand(len(rows), k, device="cuda", generator=g) < 0.5
    dA[rows] = torch.where(tiny, dA[rows].float() * 1e-10, dA[rows].float()).bfloat16()
    hA = dA.float().double().cpu().numpy()
    ties = []
    for r in rows.tolist():
        E = sum((Fraction(float(v)) for v in hA[r] if v != 0.0), Fraction(0))
        hi = float(E)
        lo = E - Fraction(hi)
        if lo != 0 and abs(lo) == abs(Fraction(np.nextafter(hi, np.inf if lo > 0 else -np.inf)) - Fraction(hi)) / 2:
            ties.append(r)
    assert len(ties) >= 5, ties
    h = FusedAbftGemm(dB)
    counts = torch.zeros(6, dtype=torch.int64, device="cuda")
    res = h(dA, counts=counts)
    torch.cuda.synchronize()
    assert int(counts[4].item()) >= len(rows) // 2, counts.tolist()
    S = torch.tensor(ties + [1, 2, 3], device="cuda")
    T_ref, _ = O.vabft_thresholds(dA[S].double().cpu().numpy(), dB.double().cpu().numpy(), h.opts.e_max, fmt="bf16")
    assert _same(res.T[S].cpu().numpy(), T_ref)
    assert int(counts[1].item()) == 0
    h.close()


def test_fp16_guard_failing_rows_integer_path(env):
    """FP16 rows that fail the exactness guard (|x| ~ 2^15.9 next to
    subnormals ~2^-24 at K = 8192): the fused kernel's integer exact sum (always exact
    for FP16: its whole range fits the 128-bit accumulator with the
    compensation provably exact) gives thresholds bit-exact against the
    reference's vabft_thresholds."""
    torch, O = env
    from paper_2602_08043_b200.fused import FusedAbftGemm
    m, k, n = 128, 8192, 512
    g = torch.Generator(device="cuda").manual_seed(41)
    A = torch.randn(m, k, device="cuda", generator=g)
    B = torch.randn(k, n, device="cuda", generator=g)
    rows = torch.arange(0, m, 5, device="cuda")
    big = torch.rand(len(rows), k, device="cuda", generator=g) < 0.02
    tiny = torch.rand(len(rows), k, device="cuda", generator=g) < 0.3
    Ar = A[rows]
    Ar = torch.where(big, Ar.sign() * 60000.0, Ar)
    Ar = torch.where(tiny, Ar.sign() * 6e-8 * torch.randint(1, 4, Ar.shape, device="cuda", generator=g), Ar)
    A[rows] = Ar
    dA, dB = A.half(), B.half()
    h = FusedAbftGemm(dB, e_max=1e-3)
    counts = torch.zeros(6, dtype=torch.int64, device="cuda")
    r = h(dA, counts=counts)
    torch.cuda.synchronize()
    assert int(counts[4].item()) >= len(rows) // 2, counts.tolist()
    S = torch.cat([rows[:20], torch.tensor([1, 2, 3], device="cuda")])
    T_ref, _ = O.vabft_thresholds(dA[S].double().cpu().numpy(), dB.double().cpu().numpy(), 1e-3, fmt="fp16")
    assert _same(r.T[S].cpu().numpy(), T_ref)
    h.close()
