"""e_max calibration on the GPU against the reference.

The reference-signature calibrate (include/vabft_cpp.hpp, bound in _core;
proj/src/calibration.cpp:88-150) runs the reference's protocol — Philox
(seed, idx) |N(1,1)| square trials, encode_and_multiply, row_sums, max
|D1| / |check1| — with every GEMM, checksum and row sum on the device EXACT
engine. Its per-size maxima, fitted model, recommended value and e_max_for
must equal the unmodified reference's calibrate() bit for bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def core_ref():
    import torch
    assert torch.cuda.is_available()
    import oracle
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    from paper_2602_08043_b200 import _core
    return _core, oracle.ref()


def _bits(x):
    return np.asarray(x, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("fmt,mode", [("bf16", "online"), ("bf16", "offline"), ("fp16", "online"),
                                      ("fp32", "offline"), ("fp64", "offline")])
def test_calibrate_matches_reference(core_ref, fmt, mode):
    core, R = core_ref
    sizes, trials, seed = [32, 64, 96], 3, 11
    F = {"bf16": core.Format.BF16, "fp16": core.Format.FP16, "fp32": core.Format.FP32, "fp64": core.Format.FP64}[fmt]
    M = core.VerifyMode.Online if mode == "online" else core.VerifyMode.Offline
    got = core.calibrate(core.PrecisionSpec.of(F), sizes, trials, seed, M)
    mx, ref = R.calibrate(fmt, sizes, trials, seed, mode=mode, dim=96)
    assert np.array_equal(_bits(got.maxima), _bits(mx))
    kind = "constant" if got.model.kind == core.EmaxModel.Kind.Constant else "sqrt_scaled"
    assert kind == ref["kind"]
    assert _bits(got.model.value) == _bits(ref["value"])
    assert _bits(got.model.scale) == _bits(ref["scale"]) and _bits(got.model.offset) == _bits(ref["offset"])
    assert _bits(got.recommended) == _bits(ref["recommended"])
    assert _bits(got.e_max_for(96)) == _bits(ref["e_max_at_dim"])
    # the Python fit on the same maxima (emax.fit_model) agrees with the C++ one
    from paper_2602_08043_b200.emax import fit_model
    pm = fit_model(sizes, list(got.maxima))
    assert pm.kind == kind and _bits(pm.scale) == _bits(got.model.scale)
