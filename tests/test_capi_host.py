"""CPU tests of the C-ABI library: it loads without a GPU, exports every
symbol include/vabft_c.h declares, and its host-side helpers (quantize,
threshold_row, resolve_e_max, aabft_sigma, localize, encode/decode_bits)
agree bit for bit with the oracle (no device compute is called here)."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def capi():
    from paper_2602_08043_b200 import _capi
    return _capi


def header_functions():
    text = open(os.path.join(ROOT, "include", "vabft_c.h")).read()
    decl = r"^(?:vabft_status|int32_t|const char\s*\*)\s*(vabft_[a-z0-9_]+)\s*\("
    return sorted(set(re.findall(decl, text, flags=re.M)))


def test_library_exports_every_header_symbol(capi):
    names = header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(capi.lib, n), f"missing export {n}"
    assert set(capi.EXPORTED) == set(names)
    assert capi.lib.vabft_api_version() == 3


def test_product_does_not_link_the_oracle():
    so = os.path.join(ROOT, "paper_2602_08043_b200", "libvabft_b200.so")
    data = open(so, "rb").read()
    assert b"libvabft_oracle" not in data and b"libvabft_ref" not in data


def test_precision_defaults(capi):
    for f, (t, kind) in {"bf16": (8, 0), "fp16": (11, 0), "fp32": (24, 3), "fp64": (53, 3)}.items():
        p = capi.precision(f)
        assert p.mantissa_bits == t and p.unit_roundoff == 2.0**-t and p.accumulation.kind == kind


def _q(capi, x, fmt):
    out = C.c_double()
    capi.check(capi.lib.vabft_quantize(x, C.byref(capi.precision(fmt)), C.byref(out)))
    return out.value


@pytest.mark.parametrize("fmt", ["bf16", "fp16", "fp32", "fp64"])
def test_host_quantize_matches_golden(capi, golden, fmt):
    xs = golden["q_x"]
    out = np.array([_q(capi, x, fmt) for x in xs])
    assert np.array_equal(out.view(np.uint64), golden[f"q_{fmt}"].view(np.uint64))


def test_quantize_errors(capi):
    with pytest.raises(capi.DomainError):
        _q(capi, math.nan, "bf16")
    p = capi.precision("fp16")
    p.overflow = 1
    out = C.c_double()
    with pytest.raises(capi.RangeError):
        capi.check(capi.lib.vabft_quantize(1e6, C.byref(p), C.byref(out)))


def test_threshold_row_and_emax(capi, port):
    out = (C.c_double * 4)()
    capi.check(capi.lib.vabft_threshold_row((C.c_double * 4)(0.0, 1.0, -1.0, 1.0), (C.c_double * 3)(0, 0, 100.0),
                                            100, 1e-3, 2.5, out))
    assert out[0] == 0.0 and out[1] == 0.0 and abs(out[3] - 0.25) < 1e-12
    rng = np.random.default_rng(1)
    for _ in range(200):
        a = [rng.normal(), 2.0, -2.0, abs(rng.normal())]
        b = list(np.abs(rng.normal(size=3)) * 10)
        n = int(rng.integers(1, 5000))
        capi.check(capi.lib.vabft_threshold_row((C.c_double * 4)(*a), (C.c_double * 3)(*b), n, 1e-3, 2.5, out))
        assert list(out) == list(port.threshold_row(a, b, n, 1e-3, 2.5))
    e = C.c_double()
    for f in ("bf16", "fp16", "fp32", "fp64"):
        for dim in (1, 77, 1024, 4096):
            capi.check(capi.lib.vabft_resolve_e_max(C.byref(capi.precision(f)), dim, C.byref(e)))
            assert e.value == port.resolve_e_max(f, dim)
    with pytest.raises(capi.InvalidArgument):
        capi.check(capi.lib.vabft_resolve_e_max(C.byref(capi.precision("fp32")), 0, C.byref(e)))


def test_aabft_sigma(capi, port):
    out = C.c_double()
    for n in (1, 512, 1024, 2048, 4096, 11008):
        for t in (8, 11, 23, 53):
            capi.check(capi.lib.vabft_aabft_sigma(n, t, 21.0, C.byref(out)))
            assert out.value == port.aabft_sigma(n, t, 21.0)


def test_localize(capi, golden):
    j = C.c_int64()
    r = C.c_double()
    for (d1, d2, n), (jj, rr) in zip(golden["loc_cases"], golden["loc_out"]):
        ok = capi.lib.vabft_localize(d1, d2, int(n), C.byref(j), C.byref(r))
        if jj < 0:
            assert not ok
        else:
            assert ok and j.value == jj and r.value == rr


@pytest.mark.parametrize("fmt", ["bf16", "fp16"])
def test_bits_every_pattern(capi, golden, fmt):
    code = capi.FORMAT_CODES[fmt]
    d = C.c_double()
    u = C.c_uint64()
    dec = golden[f"dec_{fmt}"]
    rt = golden[f"rt_{fmt}"]
    for p in range(0x10000):
        capi.check(capi.lib.vabft_decode_bits(p, code, C.byref(d)))
        assert np.float64(d.value).view(np.uint64) == dec[p].view(np.uint64)
        capi.check(capi.lib.vabft_encode_bits(d.value, code, C.byref(u)))
        assert u.value == rt[p]


def test_blockwise_thresholds_validates_before_device_work(capi):
    """vabft_blockwise_thresholds (C-ABI v3) rejects bad arguments on the host
    with the reference's invalid_argument status, before touching the device."""
    lib = capi.lib
    em = (C.c_double * 4)(1e-3, 1e-3, 1e-3, 1e-3)
    fake = C.c_void_p(16)
    bad_cases = [
        (0, 8, 8, 8, None, 0, fake, 0, 4, 4, em, 2.5, fake),     # null A
        (0, 8, 8, 8, fake, 0, fake, 0, 0, 4, em, 2.5, fake),     # tile_k = 0
        (0, 8, 8, 8, fake, 0, fake, 0, 4, 4, None, 2.5, fake),   # null e_max
        (0, 0, 8, 8, fake, 0, fake, 0, 4, 4, em, 2.5, fake),     # m = 0
        (0, 8, 8, 8, fake, 4, fake, 0, 4, 4, em, 2.5, fake),     # lda < k
        (9, 8, 8, 8, fake, 0, fake, 0, 4, 4, em, 2.5, fake),     # bad format
    ]
    for args in bad_cases:
        assert lib.vabft_blockwise_thresholds(*args, None) == capi.INVALID_ARGUMENT, args
    neg = (C.c_double * 2)(1e-3, -1.0)  # e_max < 0 on the second k-tile
    assert lib.vabft_blockwise_thresholds(0, 8, 8, 8, fake, 0, fake, 0, 4, 4, neg, 2.5, fake,
                                          None) == capi.INVALID_ARGUMENT
