"""FP16 offline false positives at large n against the reference end to end.

The C3 sweep flags a row or two per 16384 on FP16 offline N(0,1): the offline
checksum A (B r2) (position weights up to n) exceeds 65504 and saturates
(checksum.cpp:129-134, precision.cpp:153-157). For the flagged rows (and a
few clean ones) this runs the reference's own pipeline on the row slice —
encode_and_multiply (its emulated FP16 GEMM), vabft_thresholds, verify — on
the same inputs, and the reference's verify on the device's C, so each flag
is attributed: device == reference on the device's output, and the
reference's end-to-end verdict on its own output.

  python tools/fp16_offline_check.py [n] [trials] > profiles/r02_fp16_offline_check.jsonl
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (the checker)
from paper_2602_08043_b200.fused import FusedAbftGemm  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
trials = int(sys.argv[2]) if len(sys.argv) > 2 else 3
R = oracle.ref() if oracle.have_ref() else oracle.port()
for seed in range(trials):
    g_ = torch.Generator(device="cuda").manual_seed(100 + seed)
    A = torch.randn(n, n, device="cuda", generator=g_).half()
    B = torch.randn(n, n, device="cuda", generator=g_).half()
    g = FusedAbftGemm(B, mode="offline")
    r = g(A, checksums=True)
    torch.cuda.synchronize()
    det = r.detected.cpu().numpy().astype(bool)
    flagged = np.flatnonzero(det)
    S = np.unique(np.concatenate([flagged, np.arange(2)]))[:6]
    Sd = torch.from_numpy(S).cuda()
    A_s = A[Sd].double().cpu().numpy()
    B_h = B.double().cpu().numpy()
    e_max = g.opts.e_max
    T_ref, _ = R.vabft_thresholds(A_s, B_h, e_max, fmt="fp16")
    rc1, rc2 = R.blocked_row_checksums(A_s, B_h, "fp16", "offline")
    v_dev = R.verify(r.C[Sd].double().cpu().numpy(), rc1, rc2, T_ref, "fp32", "offline", accum=(2, 128))
    e = R.encode_and_multiply(A_s, B_h, "fp16", "offline")  # the reference end to end on the row slice
    v_ref = R.verify(e.c, e.row_check1, e.row_check2, T_ref, "fp16", "offline")
    for q, row in enumerate(S):
        print(json.dumps({"n": n, "seed": 100 + seed, "row": int(row), "device_flag": bool(det[row]),
                          "reference_verify_on_device_C": bool(v_dev["detected"][q]),
                          "reference_end_to_end_flag": bool(v_ref["detected"][q]),
                          "device_T_bit_exact": bool(r.T[int(row)].item() == T_ref[q]),
                          "row_check2_ref_end_to_end": float(e.row_check2[q]),
                          "saturated_row_check2": bool(abs(e.row_check2[q]) == 65504.0),
                          "flagged_rows_in_trial": int(len(flagged))}), flush=True)
    g.close()
