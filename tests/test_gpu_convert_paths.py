"""GPU parity of the conversion fast paths (ds_convert.cu) against the
oracle's COO-proxy restatement (datamove.py:208-295): bitwise.

- DIA source: the warp-group stream compaction (dia_group_counts /
  dia_group_emit) for CSR, COO and DIA targets -- ragged diagonal counts
  (1, below / at / above a warp), rows not a multiple of the group, slots
  outside the matrix, explicit and signed zeros (dropped);
- CSR source, DIA target: the order check + diagonal census in one pass
  (csr_check_mark) and the shared-memory slab fill (dia_fill_csr); rows that
  are not canonical (unsorted, duplicates) take the general path; slabs too
  wide for shared memory take the expanded-rows scatter.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2209_06478_b200 as ds  # noqa: E402
from oracle import dynsparse_oracle as O  # noqa: E402

DEV = torch.device("cuda", 0)
BIG = 2 ** 40


def host_arrays(m):
    p = m.payload if isinstance(m, ds.DynamicMatrix) else m
    if isinstance(p, ds.CsrMatrix):
        return [p.row_offsets, p.col_indices, p.values]
    if isinstance(p, ds.CooMatrix):
        return [p.row_indices, p.col_indices, p.values]
    return [p.offsets, p.values]


def oracle_arrays(m):
    if isinstance(m, O.OCsr):
        return [m.offsets, m.cols, m.vals]
    if isinstance(m, O.OCoo):
        return [m.rows, m.cols, m.vals]
    return [m.offsets, m.values]


def assert_same(dev_m, ora_m, what):
    got = [t.cpu().numpy() for t in host_arrays(dev_m)]
    want = oracle_arrays(ora_m)
    assert len(got) == len(want), what
    for g, w in zip(got, want):
        assert g.shape == np.asarray(w).shape, what
        if g.dtype.kind == "f":
            assert g.tobytes() == np.asarray(w, dtype=np.float64).tobytes(), what
        else:
            assert np.array_equal(g.astype(np.int64), np.asarray(w).astype(np.int64)), what


def random_dia(rng, nrows, ncols, nd):
    offs = np.sort(rng.choice(np.arange(-nrows + 1, ncols), size=nd, replace=False))
    vals = rng.standard_normal((nrows, nd))
    vals[rng.random(vals.shape) < 0.1] = 0.0
    vals[rng.random(vals.shape) < 0.05] = -0.0
    return offs.astype(np.int64), vals


@pytest.mark.parametrize("nrows,ncols,nd", [(1, 1, 1), (37, 37, 1), (1000, 1000, 27),
                                            (333, 500, 31), (257, 300, 32), (129, 90, 33),
                                            (70, 2000, 70)])
def test_dia_source_every_target(nrows, ncols, nd):
    rng = np.random.default_rng(nrows * 7 + nd)
    offs, vals = random_dia(rng, nrows, ncols, nd)
    src = ds.DiaMatrix(nrows, ncols, offs, vals, ds.MemorySpace.DEVICE, DEV)
    ora = O.dia(nrows, ncols, offs, vals)
    for tgt, fid in ((O.CSR, ds.FormatId.CSR), (O.COO, ds.FormatId.COO),
                     (O.DIA, ds.FormatId.DIA)):
        want = O.convert(ora, tgt, fill_limit=BIG)
        got = ds.convert(src, fid, fill_limit=BIG)
        assert_same(got, want, (nrows, ncols, nd, fid))


def test_dia_source_all_zero_and_out_of_range():
    """Every slot zero or outside the matrix: nnz == 0, row offsets all 0."""
    nrows, ncols = 100, 50
    offs = np.array([-200, 0, 60], dtype=np.int64)
    vals = np.zeros((nrows, 3))
    vals[:, 0] = 1.0     # diagonal -200: entirely outside
    vals[:, 2] = 2.0     # diagonal 60: outside (ncols 50)
    vals[:, 1] = -0.0
    src = ds.DiaMatrix(nrows, ncols, offs, vals, ds.MemorySpace.DEVICE, DEV)
    ora = O.dia(nrows, ncols, offs, vals)
    for tgt, fid in ((O.CSR, ds.FormatId.CSR), (O.COO, ds.FormatId.COO),
                     (O.DIA, ds.FormatId.DIA)):
        assert_same(ds.convert(src, fid, fill_limit=BIG), O.convert(ora, tgt, fill_limit=BIG), fid)


def test_dia_to_dia_selection_and_fill_limit():
    """DIA -> DIA keeps the diagonals holding an entry (a column selection):
    padding and -0.0 become +0.0; the default limit counts the source's
    nonzero slots; an explicit limit one slot short raises before allocation."""
    rng = np.random.default_rng(41)
    nrows, ncols = 500, 450
    offs = np.array([-600, -7, -1, 0, 3, 449, 460], dtype=np.int64)
    vals = rng.standard_normal((nrows, offs.size))
    vals[:, 2] = 0.0                      # an all-zero diagonal: dropped
    vals[::3, 3] = -0.0
    src = ds.DiaMatrix(nrows, ncols, offs, vals, ds.MemorySpace.DEVICE, DEV)
    ora = O.dia(nrows, ncols, offs, vals)
    want = O.convert(ora, O.DIA)
    got = ds.convert(src, ds.FormatId.DIA)
    assert_same(got, want, "dia->dia")
    assert list(want.offsets) == [-7, 0, 3, 449]
    with pytest.raises(ds.DiaFillOverflow):
        ds.convert(src, ds.FormatId.DIA, fill_limit=4 * nrows - 1)
    assert_same(ds.convert(src, ds.FormatId.DIA, fill_limit=4 * nrows), want, "exact limit")


def random_csr(rng, nrows, ncols, lengths, sort=True):
    offs = np.zeros(nrows + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lengths)
    cols = np.empty(offs[-1], dtype=np.int64)
    for i in range(nrows):
        c = rng.choice(ncols, size=int(lengths[i]), replace=False)
        cols[offs[i]:offs[i + 1]] = np.sort(c) if sort else c
    vals = rng.standard_normal(offs[-1])
    vals[rng.random(vals.size) < 0.05] = -0.0
    return offs, cols, vals


@pytest.mark.parametrize("nrows,ncols,maxlen", [(1, 1, 1), (300, 300, 7), (1000, 1200, 27),
                                                (513, 40, 30)])
def test_csr_to_dia_canonical(nrows, ncols, maxlen):
    rng = np.random.default_rng(nrows + maxlen)
    lengths = rng.integers(0, min(maxlen, ncols) + 1, nrows)
    offs, cols, vals = random_csr(rng, nrows, ncols, lengths)
    src = ds.CsrMatrix(nrows, ncols, offs, cols, vals, ds.MemorySpace.DEVICE, DEV)
    want = O.convert(O.csr(nrows, ncols, offs, cols, vals), O.DIA, fill_limit=BIG)
    assert_same(ds.convert(src, ds.FormatId.DIA, fill_limit=BIG), want, (nrows, ncols))


def banded_csr(rng, nrows, ncols, band):
    """Rows take a random subset of the in-range diagonals of ``band``."""
    lengths, cols = [], []
    for i in range(nrows):
        c = np.array([i + d for d in band if 0 <= i + d < ncols], dtype=np.int64)
        c = c[rng.random(c.size) < 0.8]
        if 5 <= i < 8:
            c = c[:0]                      # empty rows
        lengths.append(c.size)
        cols.append(c)
    offs = np.zeros(nrows + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lengths)
    cols = np.concatenate(cols) if cols else np.zeros(0, np.int64)
    vals = rng.standard_normal(offs[-1])
    vals[rng.random(vals.size) < 0.05] = -0.0
    return offs, cols, vals


@pytest.mark.parametrize("nrows,ncols,nbands", [(1, 1, 1), (129, 129, 5), (1000, 900, 27),
                                                (2047, 2100, 48), (300, 310, 49)])
def test_csr_to_dia_banded_slab_fill(nrows, ncols, nbands):
    """A few diagonals (the slab fits shared memory: the warp-walk fill), rows
    not a multiple of the block, empty rows, signed zeros; 49 diagonals take
    the expanded-rows scatter."""
    rng = np.random.default_rng(nrows + nbands)
    band = np.sort(rng.choice(np.arange(-60, 61), size=nbands, replace=False))
    offs, cols, vals = banded_csr(rng, nrows, ncols, band)
    src = ds.CsrMatrix(nrows, ncols, offs, cols, vals, ds.MemorySpace.DEVICE, DEV)
    want = O.convert(O.csr(nrows, ncols, offs, cols, vals), O.DIA, fill_limit=BIG)
    assert want.offsets.size <= nbands
    assert_same(ds.convert(src, ds.FormatId.DIA, fill_limit=BIG), want, (nrows, nbands))
    # a duplicate in one row: not canonical -> general path (summed)
    if offs[-1] > 2 and nrows > 10:
        cols2 = cols.copy()
        k = int(offs[nrows // 2])
        if offs[nrows // 2 + 1] - k >= 2:
            cols2[k + 1] = cols2[k]
            src = ds.CsrMatrix(nrows, ncols, offs, cols2, vals, ds.MemorySpace.DEVICE, DEV)
            want = O.convert(O.csr(nrows, ncols, offs, cols2, vals), O.DIA, fill_limit=BIG)
            assert_same(ds.convert(src, ds.FormatId.DIA, fill_limit=BIG), want, "dup")


def test_csr_to_dia_not_canonical_takes_general_path():
    rng = np.random.default_rng(11)
    nrows, ncols = 400, 400
    lengths = rng.integers(1, 12, nrows)
    offs, cols, vals = random_csr(rng, nrows, ncols, lengths, sort=False)
    cols[offs[5] + 1] = cols[offs[5]]   # a duplicate (summed)
    src = ds.CsrMatrix(nrows, ncols, offs, cols, vals, ds.MemorySpace.DEVICE, DEV)
    want = O.convert(O.csr(nrows, ncols, offs, cols, vals), O.DIA, fill_limit=BIG)
    assert_same(ds.convert(src, ds.FormatId.DIA, fill_limit=BIG), want, "unsorted")


def test_csr_to_dia_wide_slab_and_fill_limit():
    """> 6143 diagonals: the slab does not fit shared memory (expanded-rows
    scatter); the fill limit still trips before allocation."""
    rng = np.random.default_rng(12)
    nrows, ncols = 40, 9000
    lengths = np.full(nrows, 300)
    offs, cols, vals = random_csr(rng, nrows, ncols, lengths)
    src = ds.CsrMatrix(nrows, ncols, offs, cols, vals, ds.MemorySpace.DEVICE, DEV)
    want = O.convert(O.csr(nrows, ncols, offs, cols, vals), O.DIA, fill_limit=BIG)
    assert want.offsets.size > 6143
    assert_same(ds.convert(src, ds.FormatId.DIA, fill_limit=BIG), want, "wide")
    with pytest.raises(ds.DiaFillOverflow):
        ds.convert(src, ds.FormatId.DIA, fill_limit=int(want.offsets.size) * nrows - 1)


def test_stencil_round_trip_dia_csr():
    """The 27-point stencil CSR -> DIA -> CSR -> COO -> DIA: every hop bitwise
    equal to the oracle's."""
    part = ds.generate_problem(ds.GridSpec(20, 18, 16), space=ds.MemorySpace.DEVICE,
                               device=DEV).partitions[0]
    ref = O.stencil_partition(20, 18, 16).a_full
    d = ds.convert(part.a_full, ds.FormatId.DIA)
    od = O.convert(ref, O.DIA)
    assert_same(d, od, "csr->dia")
    c = ds.convert(d, ds.FormatId.CSR)
    oc = O.convert(od, O.CSR)
    assert_same(c, oc, "dia->csr")
    q = ds.convert(c, ds.FormatId.COO)
    oq = O.convert(oc, O.COO)
    assert_same(q, oq, "csr->coo")
    assert_same(ds.convert(q, ds.FormatId.DIA), O.convert(oq, O.DIA), "coo->dia")


@pytest.mark.parametrize("sort", [True, False])
def test_csr_source_to_csr_and_coo(sort):
    """Canonical CSR: copied / rows expanded in place (csr_rows_walk);
    unsorted rows: sorted through the general path."""
    rng = np.random.default_rng(21 + sort)
    nrows, ncols = 1500, 700
    lengths = rng.integers(0, 40, nrows)
    lengths[100] = 600                      # a long row (many chunks for one lane group)
    offs, cols, vals = random_csr(rng, nrows, ncols, lengths, sort=sort)
    src = ds.CsrMatrix(nrows, ncols, offs, cols, vals, ds.MemorySpace.DEVICE, DEV)
    ora = O.csr(nrows, ncols, offs, cols, vals)
    for tgt, fid in ((O.CSR, ds.FormatId.CSR), (O.COO, ds.FormatId.COO)):
        assert_same(ds.convert(src, fid, fill_limit=BIG), O.convert(ora, tgt, fill_limit=BIG),
                    (sort, fid))


@pytest.mark.parametrize("kind", ["unsorted", "repeated"])
def test_dia_source_unsorted_or_repeated_offsets(kind):
    """Offsets that are not strictly ascending: slot order is not canonical,
    so the entries take the proxy's stable sort + duplicate sums (the oracle's
    diagonal-major walk then lexsort, datamove.py:208-235)."""
    rng = np.random.default_rng(31)
    nrows, ncols = 300, 280
    offs = np.array([5, -3, 0, 40, -100, 2], dtype=np.int64)
    if kind == "repeated":
        offs = np.array([-3, 0, 0, 2, 2, 2, 40], dtype=np.int64)
    vals = rng.standard_normal((nrows, offs.size))
    vals[rng.random(vals.shape) < 0.1] = 0.0
    src = ds.DiaMatrix(nrows, ncols, offs, vals, ds.MemorySpace.DEVICE, DEV)
    ora = O.dia(nrows, ncols, offs, vals)
    for tgt, fid in ((O.CSR, ds.FormatId.CSR), (O.COO, ds.FormatId.COO),
                     (O.DIA, ds.FormatId.DIA)):
        assert_same(ds.convert(src, fid), O.convert(ora, tgt), (kind, fid))


def _row_sorted_coo(rng, nrows, ncols, lengths, dup_frac=0.1):
    rows = np.repeat(np.arange(nrows, dtype=np.int64), lengths)
    cols = rng.integers(0, ncols, rows.size)
    dup = rng.random(rows.size) < dup_frac           # duplicates inside rows
    if rows.size > 1:
        src = np.maximum(np.arange(rows.size) - 1, 0)
        same = dup & (rows == rows[src])
        cols[same] = cols[src[same]]
    vals = rng.standard_normal(rows.size)
    vals[rng.random(rows.size) < 0.02] = -0.0
    return rows, cols, vals


@pytest.mark.parametrize("case", ["short", "mixed", "long", "too_long", "empty_rows"])
def test_row_sorted_coo_segmented_sort(case):
    """Row-sorted COO with unsorted columns and duplicates takes the sort
    inside each row (warp tiles <= 128-entry rows, one CTA per longer row up
    to 16384; a longer row falls back to the LSD radix sort): canonical COO,
    CSR and the duplicate sums bitwise equal to the oracle (datamove.py:208-243)."""
    rng = np.random.default_rng({"short": 1, "mixed": 2, "long": 3, "too_long": 4,
                                 "empty_rows": 5}[case])
    nrows, ncols = 3000, 50_000
    if case == "short":
        lengths = rng.integers(0, 20, nrows)
    elif case == "mixed":
        lengths = np.minimum(nrows, np.floor(6.0 * (1 - rng.random(nrows)) ** (-1 / 1.8))).astype(int)
    elif case == "long":
        lengths = rng.integers(0, 8, nrows)
        lengths[[5, 700, 2999]] = [129, 2049, 16384]
    elif case == "too_long":
        lengths = rng.integers(0, 8, nrows)
        lengths[17] = 20_000
    else:
        lengths = np.where(rng.random(nrows) < 0.9, 0, rng.integers(1, 300, nrows))
    rows, cols, vals = _row_sorted_coo(rng, nrows, ncols, lengths)
    coo = ds.CooMatrix(nrows, ncols, rows, cols, vals, ds.MemorySpace.DEVICE, DEV)
    src = O.coo(nrows, ncols, rows, cols, vals)
    for target, name in ((ds.FormatId.COO, "coo"), (ds.FormatId.CSR, "csr")):
        got = ds.convert(coo, target)
        want = O.convert(src, O.COO if name == "coo" else O.CSR)
        assert_same(got, want, f"{case} -> {name}")
    # a CSR source with unsorted columns / duplicates: same path via its offsets
    off = np.zeros(nrows + 1, np.int64)
    np.cumsum(lengths, out=off[1:])
    csr = ds.CsrMatrix(nrows, ncols, torch.from_numpy(off.astype(np.int32)).to(DEV),
                       torch.from_numpy(cols.astype(np.int32)).to(DEV),
                       torch.from_numpy(vals).to(DEV), ds.MemorySpace.DEVICE)
    assert_same(ds.convert(csr, ds.FormatId.CSR),
                O.convert(O.csr(nrows, ncols, off, cols, vals), O.CSR), f"{case} csr src")


@pytest.mark.parametrize("shift", [0, 1, 2, 3])
def test_csr_census_quads_edges(shift):
    """The quad census (csr_census_quads): columns misaligned by 0-3 ints, a
    row longer than two row-id chunks (8192 entries), rows across 128-row
    tiles; a single duplicate / descending pair placed at every position of
    a quad, at warp (128-entry) and chunk edges and at a tile's first row
    must send the conversion down the general path (oracle-equal), while the
    same columns across a row boundary must not."""
    rng = np.random.default_rng(70 + shift)
    nrows, ncols = 400, 30000
    lengths = rng.integers(0, 40, nrows)
    lengths[130] = 20000                    # three chunks inside tile 1
    lengths[255] = 0
    offs, cols, vals = random_csr(rng, nrows, ncols, lengths)
    def conv(c, tgt):
        src = ds.CsrMatrix(nrows, ncols, torch.from_numpy(offs.astype(np.int32)).to(DEV), c,
                           torch.from_numpy(vals).to(DEV), ds.MemorySpace.DEVICE, DEV)
        return ds.convert(src, tgt, fill_limit=BIG)
    def dev_cols(cc):
        buf = torch.zeros(cc.size + 4, dtype=torch.int32, device=DEV)
        buf[shift:shift + cc.size] = torch.from_numpy(cc.astype(np.int32)).to(DEV)
        v = buf[shift:shift + cc.size]
        assert (v.data_ptr() >> 2) & 3 == ((buf.data_ptr() >> 2) + shift) & 3
        return v
    ora = O.csr(nrows, ncols, offs, cols, vals)
    for tgt, fid in ((O.CSR, ds.FormatId.CSR), (O.DIA, ds.FormatId.DIA)):
        assert_same(conv(dev_cols(cols), fid), O.convert(ora, tgt, fill_limit=BIG), (shift, fid))
    # positions: entry k's quad is (k + s) >> 2 with s the pointer's int offset
    s = (int(dev_cols(cols).data_ptr()) >> 2) & 3
    e0 = int(offs[128])
    kq0 = ((e0 + s) & ~3) - s
    L = int(offs[130])
    cand = [L + j for j in range(1, 9)] + [kq0 + 8192 + d for d in (-1, 0, 1)] \
        + [kq0 + 16384 + d for d in (0, 1)] + [kq0 + 128 * 7, kq0 + 128 * 7 + 1] \
        + [int(offs[256]) + 1, int(offs[1]) + 1]
    for k in cand:
        row = int(np.searchsorted(offs, k, side="right") - 1)
        assert offs[row] < k < offs[row + 1]          # k and k - 1 in one row
        for kind in ("swap", "dup"):
            c2 = cols.copy()
            if kind == "swap":
                c2[k - 1], c2[k] = c2[k], c2[k - 1]
                tgt, fid = O.CSR, ds.FormatId.CSR
            else:
                c2[k] = c2[k - 1]
                tgt, fid = O.DIA, ds.FormatId.DIA
            want = O.convert(O.csr(nrows, ncols, offs, c2, vals), tgt, fill_limit=BIG)
            assert_same(conv(dev_cols(c2), fid), want, (shift, k, kind))
    # a row's first column below the previous row's last: still canonical
    k = int(offs[200])
    c3 = cols.copy()
    c3[k] = 0
    c3[k:offs[201]] = np.sort(c3[k:offs[201]])
    if offs[201] - k > 1 and c3[k + 1] != 0:
        want = O.convert(O.csr(nrows, ncols, offs, c3, vals), O.CSR, fill_limit=BIG)
        got = conv(dev_cols(c3), ds.FormatId.CSR)
        assert_same(got, want, "row boundary")


@pytest.mark.parametrize("nrows,ncols,nd", [(5000, 5000, 1), (4099, 4000, 2), (3001, 3100, 7),
                                            (6000, 5990, 27), (2080, 2100, 32)])
def test_dia_source_banded_interior_groups(nrows, ncols, nd):
    """Narrow bands: most 32-row groups have every diagonal in range (the
    counts / emit interior path: 16-B loads, offsets in lanes), the first and
    last groups do not; zeros and -0.0 dropped, odd slot counts."""
    rng = np.random.default_rng(nrows + nd)
    offs = np.sort(rng.choice(np.arange(-40, 41), size=nd, replace=False)).astype(np.int64)
    vals = rng.standard_normal((nrows, nd))
    vals[rng.random(vals.shape) < 0.15] = 0.0
    vals[rng.random(vals.shape) < 0.05] = -0.0
    src = ds.DiaMatrix(nrows, ncols, offs, vals, ds.MemorySpace.DEVICE, DEV)
    ora = O.dia(nrows, ncols, offs, vals)
    for tgt, fid in ((O.CSR, ds.FormatId.CSR), (O.COO, ds.FormatId.COO),
                     (O.DIA, ds.FormatId.DIA)):
        assert_same(ds.convert(src, fid), O.convert(ora, tgt), (nrows, nd, fid))
    # DIA -> DIA with one diagonal all zero (dropped: the masked selection)
    # and with one diagonal nonzero only in the last row
    if nd > 1:
        v2 = vals.copy()
        v2[:, nd // 2] = 0.0
        v2[:, 0] = 0.0
        v2[-1, 0] = 3.0
        src = ds.DiaMatrix(nrows, ncols, offs, v2, ds.MemorySpace.DEVICE, DEV)
        want = O.convert(O.dia(nrows, ncols, offs, v2), O.DIA)
        assert_same(ds.convert(src, ds.FormatId.DIA), want, (nrows, nd, "drop"))


def _banded_rows(nrows, ncols, band, rng):
    offs = np.zeros(nrows + 1, dtype=np.int64)
    cols = []
    for i in range(nrows):
        c = np.array([i + d for d in band if 0 <= i + d < ncols], dtype=np.int64)
        cols.append(c)
        offs[i + 1] = offs[i] + c.size
    return offs, cols


def _spec_direct(src, fill_limit=-(2 ** 63)):
    """ds_convert_begin_csr_dia_spec + finish_dia through ctypes: (rc_begin,
    nd_sampled, rc_finish)."""
    import ctypes
    from paper_2209_06478_b200 import _device, _native
    lib = _native.load()
    p = _device.ptr
    job, nd = ctypes.c_void_p(), ctypes.c_int64()
    rc = lib.ds_convert_begin_csr_dia_spec(src.nrows, src.ncols, src.nnz, p(src.row_offsets),
                                           p(src.col_indices), p(src.values), fill_limit,
                                           _device.stream(DEV), ctypes.byref(job),
                                           ctypes.byref(nd))
    if rc:
        return rc, nd.value, None
    o = torch.empty(nd.value, dtype=torch.int32, device=DEV)
    v = torch.empty((src.nrows, nd.value), dtype=torch.float64, device=DEV)
    return rc, nd.value, lib.ds_convert_finish_dia(job, p(o), p(v))


def test_csr_to_dia_speculative_hit_and_miss():
    """The speculative one-pass CSR -> DIA (diagonal set from sampled 128-row
    tiles): a band present in every tile is a hit (rc 0, bitwise equal to the
    oracle); one extra diagonal only in an unsampled tile is a miss
    (DS_ERR_RETRY) and the public convert still returns the oracle's DIA
    through the census path; a sample inside the fill limit whose true set is
    not raises DiaFillOverflow; a column out of range in an unsampled tile
    raises IndexOutOfRange."""
    rng = np.random.default_rng(77)
    nrows = ncols = 128 * 600            # 600 tiles: every 2nd sampled (+ the last)
    band = [-300, -1, 0, 1, 300]
    offs, cl = _banded_rows(nrows, ncols, band, rng)
    cols = np.concatenate(cl)
    vals = rng.standard_normal(cols.size)
    vals[rng.random(cols.size) < 0.05] = -0.0
    src = ds.CsrMatrix(nrows, ncols, offs, cols, vals, ds.MemorySpace.DEVICE, DEV)
    rc, nd, rcf = _spec_direct(src)
    assert (rc, nd, rcf) == (0, 5, 0)
    want = O.convert(O.csr(nrows, ncols, offs, cols, vals), O.DIA)
    assert_same(ds.convert(src, ds.FormatId.DIA), want, "hit")
    # one entry on diagonal +777 in row 3*128+5 (tile 3: not sampled)
    r = 3 * 128 + 5
    cl2 = [c.copy() for c in cl]
    cl2[r] = np.sort(np.append(cl2[r], r + 777))
    offs2 = np.zeros(nrows + 1, np.int64)
    offs2[1:] = np.cumsum([c.size for c in cl2])
    cols2 = np.concatenate(cl2)
    vals2 = rng.standard_normal(cols2.size)
    src2 = ds.CsrMatrix(nrows, ncols, offs2, cols2, vals2, ds.MemorySpace.DEVICE, DEV)
    rc, nd, rcf = _spec_direct(src2)
    assert (rc, nd, rcf) == (0, 5, 8)
    want2 = O.convert(O.csr(nrows, ncols, offs2, cols2, vals2), O.DIA)
    assert want2.offsets.size == 6
    assert_same(ds.convert(src2, ds.FormatId.DIA), want2, "miss")
    # the sample's 5 diagonals fit the limit, the true 6 do not
    with pytest.raises(ds.DiaFillOverflow):
        ds.convert(src2, ds.FormatId.DIA, fill_limit=5 * nrows)
    # a column outside the shape in an unsampled tile
    cols3 = cols.copy()
    cols3[int(offs[r])] = ncols + 5
    src3 = ds.CsrMatrix(nrows, ncols, offs, cols3, vals, ds.MemorySpace.DEVICE, DEV)
    with pytest.raises(ds.IndexOutOfRange):
        ds.convert(src3, ds.FormatId.DIA)


def test_coo_to_dia_speculative_hit_and_miss():
    """The speculative COO -> DIA (diagonal set from 256 sampled 4096-entry
    chunks, then a checked scatter): a hit is bitwise the oracle's; an extra
    diagonal only inside an unsampled chunk is a miss (DS_ERR_RETRY from
    finish) and the public convert falls back to the census path; an
    unsorted pair in an unsampled chunk likewise."""
    import ctypes
    from paper_2209_06478_b200 import _device, _native
    rng = np.random.default_rng(78)
    nrows = ncols = 512_000                  # 2.56 M entries: 625 chunks, every 2nd sampled
    band = np.array([-700, -1, 0, 1, 700])
    rows = np.repeat(np.arange(nrows), band.size)
    cols = rows + np.tile(band, nrows)
    keep = (cols >= 0) & (cols < ncols)
    rows, cols = rows[keep], cols[keep]
    vals = rng.standard_normal(rows.size)
    vals[rng.random(rows.size) < 0.05] = -0.0

    def spec(r, c, v):
        lib = _native.load()
        p = _device.ptr
        rt, ct, vt = (torch.from_numpy(np.asarray(a, dt)).to(DEV)
                      for a, dt in ((r, np.int32), (c, np.int32), (v, np.float64)))
        job, nd = ctypes.c_void_p(), ctypes.c_int64()
        rc = lib.ds_convert_begin_coo_dia_spec(nrows, ncols, r.size, p(rt), p(ct), p(vt),
                                               -(2 ** 63), _device.stream(DEV), ctypes.byref(job),
                                               ctypes.byref(nd))
        assert rc == 0
        o = torch.empty(nd.value, dtype=torch.int32, device=DEV)
        d = torch.empty((nrows, nd.value), dtype=torch.float64, device=DEV)
        return nd.value, lib.ds_convert_finish_dia(job, p(o), p(d))

    assert spec(rows, cols, vals) == (5, 0)
    src = ds.CooMatrix(nrows, ncols, rows, cols, vals, ds.MemorySpace.DEVICE, DEV)
    assert_same(ds.convert(src, ds.FormatId.DIA),
                O.convert(O.coo(nrows, ncols, rows, cols, vals), O.DIA), "hit")
    k = 3 * 4096 + 100                        # chunk 3: not sampled
    r = int(rows[k])
    ins = int(np.searchsorted(rows, r, side="right"))   # append to row r (col r + 900)
    rows2 = np.insert(rows, ins, r)
    cols2 = np.insert(cols, ins, r + 900)
    vals2 = np.insert(vals, ins, 2.5)
    assert spec(rows2, cols2, vals2) == (5, 8)
    src2 = ds.CooMatrix(nrows, ncols, rows2, cols2, vals2, ds.MemorySpace.DEVICE, DEV)
    want2 = O.convert(O.coo(nrows, ncols, rows2, cols2, vals2), O.DIA)
    assert want2.offsets.size == 6
    assert_same(ds.convert(src2, ds.FormatId.DIA), want2, "miss")
    cols3 = cols.copy()
    cols3[k], cols3[k + 1] = cols3[k + 1], cols3[k]
    if rows[k] == rows[k + 1]:
        assert spec(rows, cols3, vals)[1] == 8
        src3 = ds.CooMatrix(nrows, ncols, rows, cols3, vals, ds.MemorySpace.DEVICE, DEV)
        assert_same(ds.convert(src3, ds.FormatId.DIA),
                    O.convert(O.coo(nrows, ncols, rows, cols3, vals), O.DIA), "unsorted")
