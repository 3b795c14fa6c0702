"""e_max models (CPU): fit_model / e_max_for against the reference's own
calibrate() (calibration.cpp:15-150) on the maxima it measured, and the
device-calibration defaults of the fused path."""
import math

import pytest

from paper_2602_08043_b200 import emax


@pytest.mark.parametrize("fmt,mode,sizes,dim", [
    ("bf16", "offline", (16, 32, 64), 64),
    ("fp16", "offline", (16, 32, 48, 64), 100),
    ("fp32", "offline", (16, 32, 64), 256),
    ("bf16", "online", (16, 32, 64), 200),
    ("fp64", "offline", (8, 16, 32), 1000),
])
def test_fit_and_e_max_for_match_reference(ref_or_port, fmt, mode, sizes, dim):
    if ref_or_port.name != "reference":
        pytest.skip("reference library not built")
    maxima, m = ref_or_port.calibrate(fmt, sizes, 3, 11, mode, dim)
    r = emax.CalibrationResult.from_maxima(fmt, mode, sizes, list(maxima), 3)
    assert r.model.kind == m["kind"]
    assert r.model.value == pytest.approx(m["value"], rel=1e-12, abs=0)
    assert r.model.scale == pytest.approx(m["scale"], rel=1e-9, abs=1e-30)
    assert r.model.offset == pytest.approx(m["offset"], rel=1e-9, abs=1e-30)
    assert r.recommended == pytest.approx(m["recommended"], rel=1e-12)
    assert r.e_max_for(dim) == pytest.approx(m["e_max_at_dim"], rel=1e-9)


def test_fit_model_rules():
    c = emax.fit_model([128, 256, 512], [1.0e-3, 1.05e-3, 0.98e-3])
    assert c.kind == "constant" and c.cv < 0.15
    s = emax.fit_model([100, 400, 1600], [1.0, 2.0, 4.0])
    assert s.kind == "sqrt_scaled" and s.scale == pytest.approx(0.1) and s.offset == pytest.approx(0.0, abs=1e-12)
    with pytest.raises(ValueError):
        emax.fit_model([1, 2], [1.0])


def test_device_defaults_cover_the_calibration():
    for key, (sizes, maxima) in emax.DEVICE_CALIBRATION.items():
        for s, mx in zip(sizes, maxima):
            e = emax.default_e_max(key[0], key[1], s)
            assert e == pytest.approx(max(1.2 * mx, 2 * emax.unit_roundoff_for(*key)))
    # monotone in K between calibrated sizes, format constants offline
    ks = [200, 700, 3000, 5000, 11008, 20000]
    es = [emax.default_e_max("bf16", "online", k) for k in ks]
    assert all(b > a for a, b in zip(es, es[1:]))
    assert emax.default_e_max("bf16", "offline", 4096) == 8e-3
    assert emax.default_e_max("fp16", "offline", 4096) == 1e-3
    assert math.isfinite(emax.resolve_run_e_max("bf16", "online", 4096))
