"""Generate golden vectors from the UNMODIFIED reference (oracle/_ref).

Run in the build container, where /root/reference exists and
`make -C oracle ref` has produced oracle/_ref/libvabft_ref.so:

    python tests/golden/make_golden.py

Writes tests/golden/golden.npz. The fixtures pin both the plain-C oracle
restatement (CPU tests) and the CUDA path (GPU tests) to the reference's
own outputs on the same seeded inputs; nothing here reads /root/reference at
test time.
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")

FMTS = ["bf16", "fp16", "fp32", "fp64"]
DISTS = ["normal:0,1", "uniform:-1,1", "truncnormal:0,1,-1,1", "normal:1e-6,1"]
SHAPES = [(8, 12, 10), (33, 70, 129), (64, 128, 96)]


def main():
    R = oracle.ref()
    g = {}
    # ---- rng: Philox KATs (test_rng.cpp:9-21) + stream draws
    g["philox_ctr"] = np.array([[0, 0, 0, 0], [0xFFFFFFFF] * 4, [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344]],
                               dtype=np.uint64)
    g["philox_key"] = np.array([[0, 0], [0xFFFFFFFF] * 2, [0xA4093822, 0x299F31D0]], dtype=np.uint64)
    g["philox_out"] = np.array([R.philox_block(c.tolist(), k.tolist()) for c, k in zip(g["philox_ctr"], g["philox_key"])],
                               dtype=np.uint64)
    g["draw_u32"] = R.draws(42, 7, 0, 1000)
    g["draw_u64"] = R.draws(42, 7, 1, 1000)
    g["draw_double"] = R.draws(42, 7, 2, 1000)
    g["draw_normal"] = R.draws(11, 3, 3, 5000)
    g["draw_below7"] = R.draws(17, 0, 4, 1000, arg=7)

    # ---- quantize: scattered doubles spanning subnormals to overflow
    rng = np.random.default_rng(101)
    xs = np.ldexp(rng.uniform(-2, 2, 3000), rng.integers(-160, 130, 3000))
    xs = np.concatenate([xs, [0.0, -0.0, 1.0 + 2**-8, 1.0 + 3 * 2**-8, 70000.0, 1e39, -1e39, 2**-133, 2**-150, 65519.9]])
    g["q_x"] = xs
    for f in FMTS:
        g[f"q_{f}"] = np.array([R.quantize(x, f) for x in xs])

    # ---- encode_and_multiply / thresholds / verify per format x mode x shape
    for f in FMTS:
        for si, (m, k, n) in enumerate(SHAPES):
            dist = DISTS[si % len(DISTS)]
            A, B = R.trial_inputs(m, k, n, f, dist, 1000 + si, FMTS.index(f))
            g[f"A_{f}_{si}"] = A
            g[f"B_{f}_{si}"] = B
            for mode in ("offline", "online"):
                e = R.encode_and_multiply(A, B, f, mode)
                key = f"{f}_{mode}_{si}"
                g[f"C_{key}"] = e.c
                g[f"Ca_{key}"] = e.c_accum
                g[f"rc1_{key}"] = e.row_check1
                g[f"rc2_{key}"] = e.row_check2
                g[f"cc1_{key}"] = e.col_check1
                g[f"cc2_{key}"] = e.col_check2
                # row sums of the verification source, default + blocked:128 strategies
                src = e.c_accum if mode == "online" else e.c
                r1, r2 = R.row_sums(src, f, mode)
                g[f"rs1_{key}"], g[f"rs2_{key}"] = r1, r2
                if f in ("bf16", "fp16"):
                    # blocked:128 row sums (the TENSOR engine's order) via the override
                    b1, b2 = R.row_sums(src, f, mode, accum=(2, 128))
                    g[f"rsb1_{key}"], g[f"rsb2_{key}"] = b1, b2
            e_max = R.resolve_e_max(f, k)
            T, s = R.vabft_thresholds(A, B, e_max)
            g[f"T_{f}_{si}"] = T
            g[f"bsum_{f}_{si}"] = s
            g[f"emax_{f}_{si}"] = np.array([e_max])
            Ta, y, dg = R.aabft_threshold(A, B, f)
            g[f"Ta_{f}_{si}"] = Ta
            g[f"ya_{f}_{si}"] = np.array([y])

    # ---- verify with planted faults (exact integer product, test_detect.cpp style)
    for mode in ("offline", "online"):
        f = "fp32"
        A, B = R.trial_inputs(16, 24, 20, f, "uniform:-1,1", 77, 0)
        e = R.encode_and_multiply(A, B, f, mode)
        src = (e.c_accum if mode == "online" else e.c).copy()
        src[2, 5] += 1.0
        src[7, 19] += -3.5
        src[9, 0] = math.nan
        src[11, 3] = math.inf
        T = np.full(16, 1e-3)
        T[4] = 0.0
        v = R.verify(src, e.row_check1, e.row_check2, T, f, mode)
        g[f"vsrc_{mode}"], g[f"vrc1_{mode}"], g[f"vrc2_{mode}"], g[f"vT_{mode}"] = src, e.row_check1, e.row_check2, T
        for kk in ("diff1", "diff2", "detected", "location", "residual"):
            g[f"v{kk}_{mode}"] = np.asarray(v[kk])

    # ---- localize
    loc_cases = np.array([[1.0, 6.0, 10], [2.0, 2.0, 10], [0.0, 1.0, 10], [1.0, 100.0, 10], [1e-300, 1e300, 10],
                          [-1.0, -6.0, 10], [1.0, 1.5, 10], [1.0, 2.5, 10], [3.0, -9.0, 10], [1e-310, 1.0, 10]])
    g["loc_cases"] = loc_cases
    g["loc_out"] = np.array([(lambda r: (r[0], r[1]) if r else (-1, -1.0))(R.localize(a, b, int(c)))
                             for a, b, c in loc_cases])

    # ---- canonical bit encodings: every 16-bit pattern
    pats = np.arange(0x10000, dtype=np.uint64)
    for f in ("bf16", "fp16"):
        dec = np.array([R.decode_bits(int(p), f) for p in pats])
        g[f"dec_{f}"] = dec
        g[f"rt_{f}"] = np.array([R.encode_bits(d, f) for d in dec], dtype=np.uint64)

    # ---- inject: fixed and random positions
    for f in FMTS:
        A, _ = R.trial_inputs(6, 7, 1, f, "normal:0,1", 3, 0, with_b=False)
        bw = 16 if f in ("bf16", "fp16") else (32 if f == "fp32" else 64)
        outs, recs = [], []
        for rep in range(12):
            bit = (rep * 5) % bw
            d = 1 + rep % 2
            X, rec = R.inject(A, f, bit, direction=d, pos=None if rep % 3 else (rep % 6, rep % 7), seed=rep, stream=1)
            outs.append(X)
            recs.append([rec["i"], rec["j"], int(rec["applied"]), rec["direction_taken"], bit, d, rep % 3])
        g[f"inj_in_{f}"] = A
        g[f"inj_out_{f}"] = np.array(outs)
        g[f"inj_rec_{f}"] = np.array(recs, dtype=np.int64)

    # ---- campaign trials (faults.cpp:181-203) and whole campaigns
    camp = []
    for mode in ("offline", "online"):
        for bit in ((9, 12) if mode == "offline" else (14, 20, 27)):
            for t in range(25):
                o = R.campaign_trial(16, 64, 16, "bf16", "normal:1e-6,1", bit, 17, t, mode=mode, method=0,
                                     e_max=8e-3 if mode == "offline" else 2e-6)
                camp.append([0 if mode == "offline" else 1, bit, t] + list(o))
    g["campaign_trials"] = np.array(camp, dtype=np.int64)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)/1e6:.2f} MB")


if __name__ == "__main__":
    main()
