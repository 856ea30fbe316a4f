"""Matrix Market ingest (host file I/O, datamove.py:302-395) -- the path that
feeds real irregular matrices to the device conversions.
Mirrors the reference's tests (test_datamove.py:284-300) and, when the
reference is mounted, compares the parsed arrays with its own reader."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from conftest import REFERENCE_SRC

import paper_2209_06478_b200 as ds


def _identity(n=4):
    offs = np.arange(n + 1, dtype=np.int64)
    return ds.CsrMatrix(n, n, offs, np.arange(n, dtype=np.int64), np.ones(n))


def test_roundtrip_identity(tmp_path):
    path = tmp_path / "eye.mtx"
    ds.write_matrix_market(_identity(), path)
    back = ds.read_matrix_market(path)
    assert isinstance(back, ds.CooMatrix) and (back.nrows, back.ncols, back.nnz) == (4, 4, 4)
    assert np.array_equal(back.row_indices, np.arange(4))
    assert np.array_equal(back.col_indices, np.arange(4))
    assert np.array_equal(back.values, np.ones(4))


def test_header_is_exact(tmp_path):
    path = tmp_path / "eye.mtx"
    ds.write_matrix_market(_identity(), path)
    assert path.read_text().splitlines()[0] == "%%MatrixMarket matrix coordinate real general"


@pytest.mark.parametrize("text, line", [
    ("%%MatrixMarket matrix array real general\n2 2\n1.0\n", 1),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1.0\n", 1),
    ("%%MatrixMarket matrix coordinate real symmetric\n1 1 1\n1 1 1.0\n", 1),
    ("%%MatrixMarket matrix coordinate real general\n2 2\n", 2),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 x\n", 3),
])
def test_malformed_files_raise_parse_error(tmp_path, text, line):
    path = tmp_path / "bad.mtx"
    path.write_text(text)
    with pytest.raises(ds.ParseError) as exc:
        ds.read_matrix_market(path)
    assert getattr(exc.value, "line", line) == line


def test_comments_integer_field_and_duplicates(tmp_path):
    path = tmp_path / "m.mtx"
    path.write_text("%%MatrixMarket matrix coordinate integer general\n% comment\n\n"
                    "3 2 4\n1 1 2\n3 2 -1\n1 1 5\n2 1 0\n")
    m = ds.read_matrix_market(path)
    assert (m.nrows, m.ncols, m.nnz) == (3, 2, 4)
    assert np.array_equal(m.row_indices, [0, 2, 0, 1])
    assert np.array_equal(m.col_indices, [0, 1, 0, 0])
    assert np.array_equal(m.values, [2.0, -1.0, 5.0, 0.0])


@pytest.mark.gpu
def test_ingest_to_device_conversion_and_spmv(tmp_path):
    """File -> host COO -> device canonicalisation / CSR / DIA -> SpMV,
    bitwise against the oracle (duplicates summed in numpy order, explicit
    zeros kept)."""
    torch = pytest.importorskip("torch")
    from oracle import dynsparse_oracle as O
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(23)
    n, nnz = 2000, 30000
    rows, cols = rng.integers(0, n, nnz), rng.integers(0, n, nnz)
    cols[: nnz // 3] = np.minimum(rows[: nnz // 3] + rng.integers(-2, 3, nnz // 3), n - 1).clip(0)
    vals = rng.standard_normal(nnz)
    vals[::97] = 0.0
    path = tmp_path / "irr.mtx"
    ds.write_matrix_market(ds.CooMatrix(n, n, rows, cols, vals), path)
    host = ds.read_matrix_market(path)
    dcoo = ds.to_device(host, dev)
    ref = O.coo(n, n, np.asarray(host.row_indices), np.asarray(host.col_indices),
                np.asarray(host.values))
    x = rng.standard_normal(n)
    for fmt, ofmt in ((ds.FormatId.CSR, O.CSR), (ds.FormatId.COO, O.COO)):
        m = ds.convert(dcoo, fmt)
        want = O.convert(ref, ofmt)
        y = ds.DenseVector.zeros(n, ds.MemorySpace.DEVICE, dev)
        ds.spmv(ds.SERIAL, m, ds.DenseVector(torch.from_numpy(x).to(dev)), y)
        yw = np.zeros(n)
        O.spmv(want, x, yw)
        assert y.data.cpu().numpy().tobytes() == yw.tobytes(), fmt


@pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference not mounted")
def test_reader_matches_reference(tmp_path):
    sys.path.insert(0, REFERENCE_SRC)
    try:
        import dynsparse as ref
    finally:
        sys.path.remove(REFERENCE_SRC)
    rng = np.random.default_rng(17)
    n, nnz = 50, 300
    path = tmp_path / "r.mtx"
    coo = ds.CooMatrix(n, n + 3, rng.integers(0, n, nnz), rng.integers(0, n + 3, nnz),
                       rng.standard_normal(nnz))
    ds.write_matrix_market(coo, path)
    ours, theirs = ds.read_matrix_market(path), ref.read_matrix_market(path)
    for a, b in (("row_indices", "row_indices"), ("col_indices", "col_indices"),
                 ("values", "values")):
        assert np.asarray(getattr(ours, a)).tobytes() == np.asarray(getattr(theirs, b)).tobytes()
