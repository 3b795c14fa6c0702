"""VABFTMAT / CSV files and verify_files against the
reference's own matrix_io (compiled into oracle/_ref) and pipeline."""
import math
import os

import numpy as np
import pytest

from paper_2602_08043_b200 import _capi, matrix_io as mio


def same(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and np.array_equal(a[~na].view(np.uint64), b[~nb].view(np.uint64))


@pytest.fixture
def ref(ref_or_port):
    if ref_or_port.name != "reference":
        pytest.skip("reference library not built")
    return ref_or_port


@pytest.mark.parametrize("fmt", ["bf16", "fp16", "fp32", "fp64"])
def test_quantize_array_matches_reference(ref_or_port, fmt):
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.normal(0, 1, 2000), rng.normal(0, 1e-6, 200), rng.normal(0, 1e4, 200),
                        [0.0, -0.0, 1e-300, -1e-42, 65519.0, 65520.0, 3.5e38, -3.4e38, 1e308, 2.0 ** -149,
                         2.0 ** -133 * 1.5, 2.0 ** -24 * 0.5, 2.0 ** -25 * 3]])
    q = mio.quantize_array(x, fmt)
    exp = np.array([ref_or_port.quantize(float(v), fmt) for v in x])
    assert same(q, exp)


@pytest.mark.parametrize("fmt", ["bf16", "fp32"])
def test_binary_and_csv_files_interoperate_with_reference(ref, tmp_path, fmt):
    rng = np.random.default_rng(2)
    X = mio.quantize_array(rng.normal(0, 1, (7, 5)), fmt)
    X[2, 3] = np.nan  # non-finite values round-trip raw (fill_values)
    X[4, 0] = -np.inf
    ours, theirs = str(tmp_path / "ours.vabft"), str(tmp_path / "theirs.vabft")
    mio.save_matrix_binary(X, fmt, ours)
    ref.save_matrix(X, fmt, theirs, binary=True)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    for p in (ours, theirs):
        v, f = mio.load_matrix_auto(p)
        w, g = ref.load_matrix(p)
        assert f == g == fmt and same(v, X) and same(w, X)
    csv_o, csv_t = str(tmp_path / "o.csv"), str(tmp_path / "t.csv")
    mio.save_matrix_csv(X, csv_o)
    ref.save_matrix(X, fmt, csv_t, binary=False)
    assert open(csv_o).read() == open(csv_t).read()
    v, f = mio.load_matrix_auto(csv_t, fmt)
    w, _ = ref.load_matrix(csv_t, fmt)
    assert same(v, w) and same(v, X)
    # CSV values off the grid are quantized on load, like the reference
    with open(str(tmp_path / "off.csv"), "w") as fh:
        fh.write("1.00390625,2.0\n3.14159,-0.1\n")
    v, _ = mio.load_matrix_auto(str(tmp_path / "off.csv"), "bf16")
    w, _ = ref.load_matrix(str(tmp_path / "off.csv"), "bf16")
    assert same(v, w)


def test_cpp_dropin_files_interoperate_with_reference(ref, tmp_path):
    core = pytest.importorskip("paper_2602_08043_b200._core")
    rng = np.random.default_rng(5)
    X = mio.quantize_array(rng.normal(0, 1, (6, 9)), "fp16")
    X[1, 1] = np.inf
    m = core.Matrix.from_numpy(np.nan_to_num(X, posinf=1.0), core.PrecisionSpec.fp16())
    m.set_raw(1, 1, float("inf"))
    for binary, name in ((True, "c.vabft"), (False, "c.csv")):
        ours, theirs = str(tmp_path / ("o_" + name)), str(tmp_path / ("t_" + name))
        (core.save_matrix_binary if binary else core.save_matrix_csv)(m, ours)
        ref.save_matrix(X, "fp16", theirs, binary=binary)
        assert open(ours, "rb").read() == open(theirs, "rb").read()
        back = core.load_matrix_auto(theirs, core.PrecisionSpec.fp16())
        assert same(back.values(), X) and back.format().format == core.Format.FP16


def test_file_errors(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"VABFTMAT\x02\x00\x00\x00")
    with pytest.raises(mio.MatrixFileError):
        mio.load_matrix_binary(str(bad))
    mio.save_matrix_binary(np.ones((3, 3)), "fp64", str(tmp_path / "ok.bin"))
    data = (tmp_path / "ok.bin").read_bytes()
    (tmp_path / "trunc.bin").write_bytes(data[:-8])
    with pytest.raises(mio.MatrixFileError, match="truncated"):
        mio.load_matrix_binary(str(tmp_path / "trunc.bin"))
    (tmp_path / "rag.csv").write_text("1,2,3\n4,5\n")
    with pytest.raises(mio.MatrixFileError, match="ragged"):
        mio.load_matrix_csv(str(tmp_path / "rag.csv"), "fp64")
    (tmp_path / "empty.csv").write_text("\n\n")
    with pytest.raises(mio.MatrixFileError, match="empty"):
        mio.load_matrix_csv(str(tmp_path / "empty.csv"), "fp64")
    with pytest.raises(mio.MatrixFileError, match="not a VABFTMAT"):
        mio.load_matrix_binary(str(tmp_path / "rag.csv"))


@pytest.mark.gpu
@pytest.mark.parametrize("fmt,mode", [("bf16", "offline"), ("fp32", "offline"), ("bf16", "online")])
def test_verify_files_matches_reference_pipeline(ref_or_port, tmp_path, fmt, mode):
    O = ref_or_port
    A, B = O.trial_inputs(40, 96, 56, fmt, "normal:1e-6,1", 9, 0)
    pa, pb, pc = str(tmp_path / "a.vabft"), str(tmp_path / "b.vabft"), str(tmp_path / "c.vabft")
    mio.save_matrix_binary(A, fmt, pa)
    mio.save_matrix_binary(B, fmt, pb)
    e = O.encode_and_multiply(A, B, fmt, mode)
    C = e.c.copy()
    C[3, 17] = mio.quantize_array(np.array([C[3, 17] + 1.0e3]), fmt)[0]  # a clear single error
    C[30, 2] = np.nan
    mio.save_matrix_binary(C, fmt, pc)
    doc, code = mio.verify_files(pa, pb, pc, fmt, mode)
    e_max = O.resolve_e_max(fmt, 96)
    T, _ = O.vabft_thresholds(A, B, e_max, 2.5, fmt)
    v = O.verify(C, e.row_check1, e.row_check2, T, fmt, mode)
    exp_rows = [int(i) for i in np.nonzero(v["detected"])[0]]
    assert code == 2 and doc["detected"] and [r["row"] for r in doc["detected_rows"]] == exp_rows
    for r in doc["detected_rows"]:
        i = r["row"]
        assert (r["diff1"] is None) == (not math.isfinite(v["diff1"][i]))
        if r["diff1"] is not None:
            assert r["diff1"] == v["diff1"][i] and r["threshold"] == T[i]
        assert r.get("location", -1) == v["location"][i]
    assert 3 in exp_rows and 30 in exp_rows
    # the clean product: nothing flagged, exit code 0
    doc0, code0 = mio.verify_files(pa, pb, None, fmt, mode)
    assert code0 == 0 and not doc0["detected"]
