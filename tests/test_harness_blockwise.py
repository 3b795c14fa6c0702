"""Experiment runners (tightness / FPR, harness.cpp:175-351) and block-wise
V-ABFT on the device, against the same computations composed from the
reference (oracle) on the same Philox trials."""
import math

import numpy as np
import pytest

from paper_2602_08043_b200 import harness


def compensated(row):
    s = c = 0.0
    for x in row:
        t = s + x
        c += ((s - t) + x) if abs(s) >= abs(x) else ((x - t) + s)
        s = t
    return s + c


def test_trial_operands_are_the_reference_trials(ref_or_port):
    pytest.importorskip("paper_2602_08043_b200._core")
    for fmt, dist in [("fp32", "uniform:-1,1"), ("bf16", "normal:1e-6,1"), ("fp64", "truncnormal:0,1,-1,1")]:
        cfg = harness.ExperimentConfig(precision=fmt, dist=dist, m=5, k=7, n=3, seed=12)
        for t in (0, 3):
            a, b = harness.trial_operands(cfg, t)
            A, B = ref_or_port.trial_inputs(5, 7, 3, fmt, dist, 12, t)
            assert np.array_equal(a, A) and np.array_equal(b, B)


def test_compensated_sum_rows():
    rng = np.random.default_rng(0)
    x = rng.normal(0, 1, (6, 50)) * np.logspace(-8, 8, 50)
    got = harness.compensated_sum_rows(x)
    assert all(got[i] == compensated(x[i]) for i in range(6))


@pytest.mark.gpu
@pytest.mark.parametrize("fmt,mode", [("fp32", "offline"), ("fp64", "offline"), ("bf16", "online")])
def test_tightness_and_fpr_match_reference_composition(ref_or_port, fmt, mode):
    O = ref_or_port
    cfg = harness.ExperimentConfig(precision=fmt, dist="normal:1e-6,1", m=16, k=64, n=24, trials=3, seed=4,
                                   mode=mode, methods=["vabft", "aabft-fixed-y", "aabft-computed-y"])
    doc = harness.run_tightness(cfg)
    fpr = harness.run_fpr(cfg)
    e_max = doc["config"]["e_max"]["value"]
    assert e_max == O.resolve_e_max(fmt, 64)
    means, thr_means, unc = [], {m: [] for m in cfg.methods}, {m: 0 for m in cfg.methods}
    for t in range(cfg.trials):
        A, B = O.trial_inputs(16, 64, 24, fmt, "normal:1e-6,1", 4, t)
        e = O.encode_and_multiply(A, B, fmt, mode)
        src = e.c_accum if mode == "online" else e.c
        if fmt == "fp64":
            actual = np.array([abs(math.fsum([e.row_check1[i]] + [-x for x in src[i]])) for i in range(16)])
        else:
            actual = np.array([abs(e.row_check1[i] - compensated(src[i])) for i in range(16)])
        means.append(harness.seq_mean(actual))
        for m in cfg.methods:
            if m == "vabft":
                T = O.vabft_thresholds(A, B, e_max, 2.5, fmt)[0]
            else:
                T = O.aabft_threshold(A, B, fmt, computed=(m == "aabft-computed-y"),
                                      fixed_y=21.0 if m == "aabft-fixed-y" else None)[0]
            thr_means[m].append(harness.seq_mean(T))
            unc[m] += int((actual > T).sum())
    assert doc["actual"]["per_trial_mean"] == means
    for m in cfg.methods:
        assert doc["methods"][m]["per_trial_mean_threshold"] == thr_means[m]
        assert doc["methods"][m]["rows_not_covered"] == unc[m]
    assert fpr["methods"]["vabft"]["false_positive_rows"] == 0


@pytest.mark.gpu
def test_blockwise_matches_reference_on_slices(ref_or_port):
    from paper_2602_08043_b200 import blockwise
    O = ref_or_port
    A, B = O.trial_inputs(16, 64, 24, "bf16", "normal:1e-6,1", 8, 0)
    T = blockwise.blockwise_thresholds(A, B, "bf16", tile_k=32, tile_n=8, e_max=8e-3)
    assert T.shape == (16, 3)
    for jb, j0 in enumerate((0, 8, 16)):
        exp = sum(O.vabft_thresholds(np.ascontiguousarray(A[:, k0:k0 + 32]),
                                     np.ascontiguousarray(B[k0:k0 + 32, j0:j0 + 8]), 8e-3, 2.5, "bf16")[0]
                  for k0 in (0, 32))
        assert np.array_equal(T[:, jb], exp)
    e = O.encode_and_multiply(A, B, "bf16", "offline")
    C = e.c.copy()
    C[5, 13] = 512.0  # a single error, on the BF16 grid
    v = blockwise.blockwise_verify(A, B, C, "bf16", "offline", tile_k=32, tile_n=8, e_max=8e-3)
    assert v.detected[5] and v.location[5] == 13 and v.block_detected[5].tolist() == [False, True, False]
    assert not v.detected[np.arange(16) != 5].any()
    # block 1 verdicts are the reference's verify on that slice
    e1 = O.encode_and_multiply(A, np.ascontiguousarray(B[:, 8:16]), "bf16", "offline")
    r = O.verify(np.ascontiguousarray(C[:, 8:16]), e1.row_check1, e1.row_check2, T[:, 1], "bf16", "offline")
    assert np.array_equal(v.diff1[:, 1], r["diff1"])


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["bf16", "fp32", "fp16", "fp64"])
def test_blockwise_device_kernels_equal_slice_composition(fmt):
    """csrc/blockwise.cu (three launches) equals the slice-by-slice
    composition of the reference's vabft_thresholds (threshold_vabft.cpp:54-61)
    bit for bit, with ragged last k-tile and column block, e_max per k-tile
    from the format model."""
    import torch

    from paper_2602_08043_b200 import blockwise
    g = np.random.default_rng(7)
    m, k, n = 96, 1000, 600
    A = g.standard_normal((m, k))
    B = g.standard_normal((k, n)) * 0.05 + 0.01
    if fmt in ("bf16", "fp16"):
        dt = torch.bfloat16 if fmt == "bf16" else torch.float16
        A = torch.from_numpy(A).to(dt).double().numpy()
        B = torch.from_numpy(B).to(dt).double().numpy()
    elif fmt == "fp32":
        A, B = A.astype(np.float32).astype(np.float64), B.astype(np.float32).astype(np.float64)
    Td = blockwise.blockwise_thresholds(A, B, fmt, tile_k=384, tile_n=128)
    Ts = blockwise.blockwise_thresholds(A, B, fmt, tile_k=384, tile_n=128, engine="slices")
    assert Td.shape == (m, 5)
    assert np.array_equal(Td.view(np.uint64), Ts.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["bf16", "fp32"])
def test_fused_kernel_verifies_against_given_blockwise_thresholds(ref_or_port, fmt):
    """Threshold method 3 (vabft_fused_opts.t_in): the fused kernel verifies
    a column block of C against the block-wise thresholds T[:, J]; its
    verdicts, differences and located column equal the reference's verify
    (detect.cpp:19-55) on the device's own accumulator with the same T, and a
    planted accumulator fault is located. blockwise_verify_fused runs all
    blocks: clean rows give no detections."""
    import torch

    from paper_2602_08043_b200 import blockwise
    from paper_2602_08043_b200.fused import FusedAbftGemm
    O = ref_or_port
    m, k, n, tk, tn = 256, 2048, 512, 1024, 256
    dt = torch.bfloat16 if fmt == "bf16" else torch.float32
    g0 = torch.Generator(device="cuda").manual_seed(11)
    A = torch.randn(m, k, device="cuda", generator=g0).to(dt)
    B = torch.randn(k, n, device="cuda", generator=g0).to(dt)
    T = blockwise.blockwise_thresholds_device(A, B, fmt, tile_k=tk, tile_n=tn)
    Ts = blockwise.blockwise_thresholds(A.double().cpu().numpy(), B.double().cpu().numpy(), fmt, tk, tn,
                                        engine="slices")
    assert np.array_equal(T.cpu().numpy().view(np.uint64), Ts.view(np.uint64))
    jb, j0, j1 = 1, 256, 512
    bj = B[:, j0:j1] if fmt == "bf16" else B[:, j0:j1].contiguous()
    g = FusedAbftGemm(bj, mode="online")
    col = torch.full((m,), -1, dtype=torch.int32, device="cuda")
    bit = torch.zeros(m, dtype=torch.int32, device="cuda")
    col[9], bit[9] = 77, 29
    acc = torch.empty(m, j1 - j0, dtype=torch.float32, device="cuda") if fmt == "bf16" else None
    r = g(A, t_in=T[:, jb], checksums=True, accum_out=acc,
          faults={"col": col, "bit": bit, "dir": torch.zeros(m, dtype=torch.int32, device="cuda")})
    torch.cuda.synchronize()
    assert np.array_equal(r.T.cpu().numpy(), T[:, jb].cpu().numpy())
    src = (acc if fmt == "bf16" else r.C).double().cpu().numpy()
    v = O.verify(src, r.row_check1.cpu().numpy(), r.row_check2.cpu().numpy(), T[:, jb].cpu().numpy(),
                 "fp32" if fmt == "bf16" else fmt, "offline" if fmt == "bf16" else "online", accum=(2, 128))
    assert np.array_equal(v["detected"], r.detected.cpu().numpy().astype(bool))
    assert np.array_equal(v["diff1"].view(np.uint64), r.diff1.cpu().numpy().view(np.uint64))
    assert np.array_equal(v["location"], r.location.cpu().numpy())
    assert bool(r.detected[9].item()) and int(r.location[9].item()) == 77
    g.close()
    fv = blockwise.blockwise_verify_fused(A, B, fmt, "online", tile_k=tk, tile_n=tn)
    torch.cuda.synchronize()
    assert not bool(fv.detected.any().item())
    assert int((fv.location >= 0).sum().item()) == 0


@pytest.mark.gpu
def test_blockwise_fused_graph_replay_equals_eager():
    """BlockwiseFusedGemm's CUDA-graph replay (the per-block launches
    recorded once per M) gives the same C, thresholds and verdicts as the
    eager per-block calls, on two different activations, with a planted
    single error found at its global column."""
    import torch

    from paper_2602_08043_b200 import blockwise
    g0 = torch.Generator(device="cuda").manual_seed(5)
    m, k, n = 512, 2048, 768
    B = torch.randn(k, n, device="cuda", generator=g0).bfloat16()
    eager = blockwise.BlockwiseFusedGemm(B, "bf16", "online", 1024, 256, graphs=False)
    graph = blockwise.BlockwiseFusedGemm(B, "bf16", "online", 1024, 256)
    for seed in (1, 2):
        A = torch.randn(m, k, device="cuda", generator=torch.Generator(device="cuda").manual_seed(seed)).bfloat16()
        ce, cg = torch.zeros(6, dtype=torch.int64, device="cuda"), torch.zeros(6, dtype=torch.int64, device="cuda")
        re, rg = eager(A, counts=ce), graph(A, counts=cg)
        torch.cuda.synchronize()
        assert torch.equal(re.C.view(torch.int16), rg.C.view(torch.int16))
        assert torch.equal(re.thresholds, rg.thresholds)
        assert torch.equal(re.block_detected, rg.block_detected)
        assert torch.equal(re.diff1, rg.diff1)
        assert torch.equal(ce, cg) and int(cg[0].item()) == m * 3 and int(cg[1].item()) == 0
    eager.close()
    graph.close()


def test_tile_emax_forms():
    """e_max per k-tile: one value for all tiles, one per tile (checked
    against the tile count), or the format model at dim = |kt|."""
    from paper_2602_08043_b200 import _capi, blockwise
    assert blockwise._tile_emax("bf16", 1000, 384, 1e-3).tolist() == [1e-3] * 3
    assert blockwise._tile_emax("bf16", 1000, 384, [1e-3, 2e-3, 3e-3]).tolist() == [1e-3, 2e-3, 3e-3]
    with pytest.raises(_capi.InvalidArgument):
        blockwise._tile_emax("bf16", 1000, 384, [1e-3, 2e-3])
    em = blockwise._tile_emax("fp32", 1000, 384, None)
    assert em.shape == (3,) and (em > 0).all()
