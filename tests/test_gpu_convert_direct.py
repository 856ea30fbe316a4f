"""GPU parity of the one-pass canonical conversions (ds_convert_direct:
csr_census_quads<.., COPY> and coo_direct_kernel) against the oracle's
COO-proxy restatement (datamove.py:208-295): bitwise.

A canonical COO / CSR source ((row, col) strictly increasing) goes to a COO
/ CSR target in one pass -- the C entry reports done = 1; anything else
(unsorted, duplicates, rows decreasing, misaligned arrays) reports done = 0
and the Python convert falls back to begin / finish, whose result must still
be the oracle's.  Ragged tails (nnz % 4), empty leading / trailing / interior
rows (the offsets written at row changes), signed zeros, and an index out of
range (IndexOutOfRange, like begin_*).
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2209_06478_b200 as ds  # noqa: E402
from paper_2209_06478_b200 import _device, _native  # noqa: E402
from oracle import dynsparse_oracle as O  # noqa: E402

DEV = torch.device("cuda", 0)


def canonical_coo(rng, nrows, ncols, nnz, empty_head=0, empty_tail=0):
    lo, hi = empty_head, nrows - empty_tail
    keys = np.unique(rng.integers(lo * ncols, hi * ncols, nnz))
    rows, cols = keys // ncols, keys % ncols
    vals = rng.standard_normal(keys.size)
    vals[rng.random(keys.size) < 0.1] = -0.0
    vals[rng.random(keys.size) < 0.05] = 0.0
    return rows.astype(np.int64), cols.astype(np.int64), vals


def direct(src_fmt, tgt, nrows, ncols, a0, a1, v, nnz):
    lib = _native.load()
    n0 = nnz if tgt == ds.FormatId.COO else nrows + 1
    o0 = torch.empty(n0, dtype=torch.int32, device=DEV)
    o1 = torch.empty(nnz, dtype=torch.int32, device=DEV)
    ov = torch.empty(nnz, dtype=torch.float64, device=DEV)
    done = ctypes.c_int32(-1)
    p = _device.ptr
    rc = lib.ds_convert_direct(int(src_fmt), int(tgt), nrows, ncols, nnz, p(a0), p(a1), p(v),
                               p(o0), p(o1), p(ov), _device.stream(DEV), ctypes.byref(done))
    return rc, done.value, (o0, o1, ov)


def same(got, want):
    g0, g1, gv = (t.cpu().numpy() for t in got)
    w0 = want.rows if isinstance(want, O.OCoo) else want.offsets
    return (np.array_equal(g0.astype(np.int64), np.asarray(w0, np.int64))
            and np.array_equal(g1.astype(np.int64), np.asarray(want.cols, np.int64))
            and gv.tobytes() == np.asarray(want.vals, np.float64).tobytes())


def i32(a):
    return torch.from_numpy(np.asarray(a, np.int32)).to(DEV)


def f64(a):
    return torch.from_numpy(np.asarray(a, np.float64)).to(DEV)


@pytest.mark.parametrize("nrows,ncols,nnz,head,tail", [
    (1, 1, 1, 0, 0), (1, 50, 7, 0, 0), (9, 9, 30, 2, 3), (300, 200, 4001, 0, 0),
    (1000, 37, 5002, 17, 40), (4097, 4097, 40003, 1, 1), (70000, 30, 100000, 0, 5000)])
def test_direct_canonical_sources(nrows, ncols, nnz, head, tail):
    rng = np.random.default_rng(nrows + nnz)
    r, c, v = canonical_coo(rng, nrows, ncols, nnz, head, tail)
    n = r.size
    ocoo = O.coo(nrows, ncols, r, c, v)
    ocsr = O.convert(ocoo, O.CSR)
    offs = np.asarray(ocsr.offsets)
    for src_fmt, a0 in ((ds.FormatId.COO, i32(r)), (ds.FormatId.CSR, i32(offs))):
        for tgt, want in ((ds.FormatId.COO, O.convert(ocoo, O.COO)),
                          (ds.FormatId.CSR, ocsr)):
            rc, done, out = direct(src_fmt, tgt, nrows, ncols, a0, i32(c), f64(v), n)
            assert rc == 0 and done == 1, (src_fmt, tgt)
            assert same(out, want), (src_fmt, tgt, nrows, n)
    # the public convert takes the same path and agrees
    src = ds.CooMatrix(nrows, ncols, r, c, v, ds.MemorySpace.DEVICE, DEV)
    got = ds.convert(src, ds.FormatId.CSR)
    assert same((got.row_offsets, got.col_indices, got.values), ocsr)


@pytest.mark.parametrize("kind", ["swap", "dup", "row_down", "first_quad", "last"])
@pytest.mark.parametrize("src_fmt", [ds.FormatId.COO, ds.FormatId.CSR])
def test_direct_not_canonical_falls_back(kind, src_fmt):
    rng = np.random.default_rng(5)
    nrows, ncols = 500, 400
    r, c, v = canonical_coo(rng, nrows, ncols, 6003)
    n = r.size
    k = {"swap": n // 2 + 1, "dup": n // 3 + 2, "row_down": n // 2 + 3, "first_quad": 1,
         "last": n - 1}[kind]
    while r[k] != r[k - 1] and kind in ("swap", "dup", "first_quad", "last"):
        k += 1 if kind != "last" else -1
    r2, c2 = r.copy(), c.copy()
    if kind in ("swap", "first_quad", "last"):
        c2[k - 1], c2[k] = c2[k], c2[k - 1]
    elif kind == "dup":
        c2[k] = c2[k - 1]
    else:   # a row index below the previous entry's (COO only: a CSR row order is implied)
        if src_fmt == ds.FormatId.CSR:
            pytest.skip("CSR rows cannot decrease")
        r2[k] = r2[k - 1] - 1
    ora = O.coo(nrows, ncols, r2, c2, v)
    if src_fmt == ds.FormatId.COO:
        a0 = i32(r2)
        src = ds.CooMatrix(nrows, ncols, r2, c2, v, ds.MemorySpace.DEVICE, DEV)
    else:
        offs = np.zeros(nrows + 1, np.int64)
        np.add.at(offs, r2 + 1, 1)
        offs = np.cumsum(offs)
        a0 = i32(offs)
        src = ds.CsrMatrix(nrows, ncols, offs, c2, v, ds.MemorySpace.DEVICE, DEV)
        ora = O.csr(nrows, ncols, offs, c2, v)
    for tgt, otgt in ((ds.FormatId.COO, O.COO), (ds.FormatId.CSR, O.CSR)):
        rc, done, _ = direct(src_fmt, tgt, nrows, ncols, a0, i32(c2), f64(v), n)
        assert rc == 0 and done == 0, (kind, tgt)
        got = ds.convert(src, tgt)
        want = O.convert(ora, otgt)
        arrs = ((got.row_indices if tgt == ds.FormatId.COO else got.row_offsets),
                got.col_indices, got.values)
        assert same(arrs, want), (kind, src_fmt, tgt)


def test_direct_misaligned_and_index_errors():
    rng = np.random.default_rng(8)
    nrows, ncols = 200, 150
    r, c, v = canonical_coo(rng, nrows, ncols, 3001)
    n = r.size
    # columns starting 4 bytes past an allocation: not applicable (done = 0),
    # the public convert still agrees with the oracle through begin / finish
    cbuf = torch.zeros(n + 1, dtype=torch.int32, device=DEV)
    cbuf[1:] = i32(c)
    rc, done, _ = direct(ds.FormatId.COO, ds.FormatId.CSR, nrows, ncols, i32(r), cbuf[1:], f64(v), n)
    assert rc == 0 and done == 0
    src = ds.CooMatrix(nrows, ncols, i32(r), cbuf[1:], f64(v), ds.MemorySpace.DEVICE, DEV)
    got = ds.convert(src, ds.FormatId.CSR)
    assert same((got.row_offsets, got.col_indices, got.values),
                O.convert(O.coo(nrows, ncols, r, c, v), O.CSR))
    # a column outside the shape: IndexOutOfRange from both sources
    c_bad = c.copy()
    c_bad[n // 2] = ncols
    rc, done, _ = direct(ds.FormatId.COO, ds.FormatId.COO, nrows, ncols, i32(r), i32(c_bad),
                         f64(v), n)
    assert rc == 7 and done == 0
    with pytest.raises(ds.IndexOutOfRange):
        ds.convert(ds.CooMatrix(nrows, ncols, r, c_bad, v, ds.MemorySpace.DEVICE, DEV),
                   ds.FormatId.CSR)
    offs = np.asarray(O.convert(O.coo(nrows, ncols, r, c, v), O.CSR).offsets)
    with pytest.raises(ds.IndexOutOfRange):
        ds.convert(ds.CsrMatrix(nrows, ncols, offs, c_bad, v, ds.MemorySpace.DEVICE, DEV),
                   ds.FormatId.COO)


def test_direct_at_192_cubed():
    """The 192^3 partition (189 M entries): CSR -> COO -> CSR through the
    one-pass path, bitwise round trip and against the generator's CSR."""
    part = ds.generate_partition(ds.GridSpec(192, 192, 192), 0, space=ds.MemorySpace.DEVICE,
                                 device=DEV)
    a = part.a_full
    coo = ds.convert(a, ds.FormatId.COO)
    back = ds.convert(coo, ds.FormatId.CSR)
    assert torch.equal(back.row_offsets, a.row_offsets)
    assert torch.equal(back.col_indices, a.col_indices)
    assert torch.equal(back.values.view(torch.int64), a.values.view(torch.int64))
    # COO rows: row i repeated (offsets[i+1] - offsets[i]) times
    counts = (a.row_offsets[1:] - a.row_offsets[:-1]).long()
    rows = torch.repeat_interleave(torch.arange(a.nrows, device=DEV, dtype=torch.int32), counts)
    assert torch.equal(coo.row_indices, rows)
    assert torch.equal(coo.col_indices, a.col_indices)
