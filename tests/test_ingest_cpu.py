"""Tensor-file ingest (tensor.py:188-327) through this package, CPU suite.

The %rescalk-coo loader is the native parser in librescal_b200
(csrc/ingest.cpp); it must return exactly what the reference's loader
returns — canonical CSR arrays — and raise the reference's DataError texts.
The expected outputs in tests/golden/coo_ingest.npz were produced by the
reference itself (tests/golden/make_golden.py, case 16). No GPU is used.
"""
import os

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden

rk = pytest.importorskip("paper_2202_09512_b200")


def _write(tmp_path, name, text):
    p = os.path.join(tmp_path, name + ".coo")
    with open(p, "w", encoding="utf-8") as f:
        f.write(text)
    return p


@pytest.mark.parametrize("name", ["saved", "messy"])
def test_coo_load_matches_reference(tmp_path, name):
    g = golden("coo_ingest")
    x = rk.load_tensor(_write(tmp_path, name, str(g[f"{name}_text"])))
    assert x.n == int(g[f"{name}_n"])
    for t, s in enumerate(x.slices):
        np.testing.assert_array_equal(s.indptr, g[f"{name}_indptr{t}"])
        np.testing.assert_array_equal(s.indices, g[f"{name}_indices{t}"])
        np.testing.assert_array_equal(s.data, g[f"{name}_data{t}"])
        assert s.data.dtype == np.float64


@pytest.mark.parametrize("name", ["bad_header", "bad_fields", "bad_relation", "bad_index", "bad_negative",
                                  "bad_count", "bad_float"])
def test_coo_errors_match_reference(tmp_path, name):
    g = golden("coo_ingest")
    with pytest.raises(rk.DataError) as ei:
        rk.load_tensor(_write(tmp_path, name, str(g[f"{name}_text"])))
    assert str(ei.value) == str(g[f"{name}_error"])


def test_coo_round_trip_and_first_error_wins(tmp_path):
    rng = np.random.default_rng(5)
    slices = [sp.random(40, 40, density=0.1, random_state=rng, format="csr") for _ in range(3)]
    x = rk.SparseRelTensor(slices)
    p = os.path.join(tmp_path, "rt.coo")
    rk.save_tensor(x, p)
    y = rk.load_tensor(p)
    for a, b in zip(x.slices, y.slices):
        assert (a != b).nnz == 0
        np.testing.assert_array_equal(a.data, b.data)
    # two bad lines far apart (different parser chunks): the first one is reported
    body = "".join(f"0 {i % 7} {i % 5} 1.0\n" for i in range(200000))
    head = body[:1000].rsplit("\n", 1)[0] + "\n"
    text = "%rescalk-coo 7 1 200002\n" + head + "0 9 0 1.0\n" + body[len(head):] + "0 0 0 -1.0\n"
    bad_line = 2 + head.count("\n")
    with pytest.raises(rk.DataError, match=rf"^line {bad_line}: index \(9,0\) out of bounds$"):
        rk.load_tensor(_write(tmp_path, "two_errors", text))


def test_dense_and_matrix_formats_round_trip(tmp_path):
    x = rk.RelTensor(np.random.default_rng(1).random((2, 5, 5)).astype(np.float32))
    p = os.path.join(tmp_path, "x.rsk")
    rk.save_tensor(x, p)
    with open(p, "rb") as f:
        assert f.read(4) == b"RSK1"
    y = rk.load_tensor(p)
    assert y.slices.dtype == np.float32
    np.testing.assert_array_equal(x.slices, y.slices)
    a = np.arange(12.0).reshape(3, 4)
    pm = os.path.join(tmp_path, "a.rskm")
    rk.save_matrix(a, pm)
    np.testing.assert_array_equal(rk.load_matrix(pm), a)
    with open(p, "r+b") as f:
        f.seek(0, 2)
        f.write(b"\0")
    with pytest.raises(rk.DataError, match="dimension mismatch"):
        rk.load_tensor(p)
