"""GPU parity of the row-sorted COO SpMV (ds_coo.cu coo_pipe) against the
oracle's np.bincount restatement (kernels.py:143-163): bitwise.

Shapes that hit every branch of the pipeline: rows split across tiles and
across CTA ranges (carries), rows of exactly 27 entries, one row longer than a whole CTA range, runs of
absent rows (written as +0.0 by their owner), more rows than entries,
duplicates and signed zeros, spmv_add, and sizes that are not multiples of
the 16-byte bulk-copy granule (hand-copied tails).
"""

from __future__ import annotations

import ctypes
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_2209_06478_b200 import _device, _native  # noqa: E402
from oracle import dynsparse_oracle as O  # noqa: E402

DEV = torch.device("cuda", 0)


def run(nrows, ncols, rows, cols, vals, x, y0, accumulate, planned=True):
    """ds_spmv_coo_sorted with the longest row from ds_coo_max_run (the
    pipeline when it is <= 27), or plain ds_spmv_coo (warp kernel)."""
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(DEV)  # noqa: E731
    r, c, v, xt = t(rows, np.int32), t(cols, np.int32), t(vals, np.float64), t(x, np.float64)
    y = t(y0, np.float64)
    st = _device.stream(DEV)
    if planned:
        mr = ctypes.c_int32(-1)
        _native.call("ds_coo_max_run", rows.size, r.data_ptr(), ctypes.byref(mr), st)
        lens = np.bincount(rows, minlength=nrows) if rows.size else np.zeros(1, np.int64)
        assert mr.value == int(lens.max())
        _native.call("ds_spmv_coo_sorted", nrows, ncols, rows.size, r.data_ptr(), c.data_ptr(),
                     v.data_ptr(), mr.value, xt.data_ptr(), y.data_ptr(), int(accumulate), st)
    else:
        _native.call("ds_spmv_coo", nrows, ncols, rows.size, r.data_ptr(), c.data_ptr(),
                     v.data_ptr(), 1, xt.data_ptr(), y.data_ptr(), int(accumulate), st)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def want(nrows, ncols, rows, cols, vals, x, y0, accumulate):
    m = O.coo(nrows, ncols, rows.astype(np.int64), cols.astype(np.int64), vals)
    y = y0.copy()
    (O.spmv_add if accumulate else O.spmv)(m, x, y)
    return y


def sorted_coo(rng, nrows, ncols, lengths):
    rows = np.repeat(np.arange(nrows, dtype=np.int64), lengths)
    cols = rng.integers(0, ncols, rows.size)          # duplicates allowed, unordered cols
    vals = rng.standard_normal(rows.size)
    vals[rng.random(rows.size) < 0.02] = -0.0
    return rows, cols, vals


CASES = {
    "stencil_like": lambda rng: (20000, 20000, rng.integers(20, 28, 20000)),
    "ragged_with_gaps": lambda rng: (30011, 5000, np.where(rng.random(30011) < 0.3, 0,
                                                              rng.integers(1, 40, 30011))),
    "sparse_rows": lambda rng: (400_000, 1000, (rng.random(400_000) < 0.01).astype(np.int64) * 3),
    "power_law": lambda rng: (50_000, 50_000, np.minimum(
        50_000, np.floor(6.0 * (1 - rng.random(50_000)) ** (-1 / 1.8))).astype(np.int64)),
    "tiny": lambda rng: (7, 5, np.array([0, 3, 1, 0, 0, 2, 1])),
    "rows_up_to_27": lambda rng: (9000, 4000, rng.integers(0, 28, 9000)),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_coo_pipe_bitwise(name):
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    nrows, ncols, lengths = CASES[name](rng)
    rows, cols, vals = sorted_coo(rng, nrows, ncols, lengths)
    x = rng.standard_normal(ncols)
    for acc in (False, True):
        y0 = rng.standard_normal(nrows)
        y0[::7] = -0.0
        ref = want(nrows, ncols, rows, cols, vals, x, y0, acc).tobytes()
        for planned in (True, False):
            got = run(nrows, ncols, rows, cols, vals, x, y0, acc, planned)
            assert got.tobytes() == ref, (name, acc, planned)


def test_coo_pipe_giant_row_and_odd_tail():
    """One row spanning several CTA ranges, entries count % 4 != 0, leading
    and trailing absent rows."""
    rng = np.random.default_rng(11)
    nrows, ncols = 1000, 3000
    lengths = np.zeros(nrows, dtype=np.int64)
    lengths[10] = 3
    lengths[500] = 700_001
    lengths[501:990] = rng.integers(0, 5, 489)
    rows, cols, vals = sorted_coo(rng, nrows, ncols, lengths)
    x = rng.standard_normal(ncols)
    for acc in (False, True):
        y0 = rng.standard_normal(nrows)
        got = run(nrows, ncols, rows, cols, vals, x, y0, acc)
        assert got.tobytes() == want(nrows, ncols, rows, cols, vals, x, y0, acc).tobytes(), acc


def test_coo_long_runs_split_bitwise():
    """Rows longer than the long-run threshold are summed by their own kernel
    on a side stream while the warp kernel skips them (descriptor path): runs
    at the start, back to back, spanning many warp chunks, at the end."""
    import paper_2209_06478_b200 as ds
    from paper_2209_06478_b200 import kernels as K_
    thr = int(_native.load().ds_coo_long_run_threshold())
    rng = np.random.default_rng(31)
    nrows, ncols = 3000, 40000
    lengths = rng.integers(0, 30, nrows)
    lengths[0] = thr + 1            # first row long
    lengths[10] = 3 * thr + 7       # two long rows back to back
    lengths[11] = 20000             # spans several 4096-entry chunks
    lengths[1500] = thr + 1
    lengths[2999] = 2 * thr + 5     # last row long
    lengths[[5, 6, 2000, 2001]] = 0
    rows, cols, vals = sorted_coo(rng, nrows, ncols, lengths)
    x = rng.standard_normal(ncols)
    a = ds.CooMatrix(nrows, ncols, rows, cols, vals, ds.MemorySpace.DEVICE, DEV)
    runs, cnt = K_.coo_long_runs(a)
    assert cnt == 5
    r = runs.cpu().numpy().reshape(-1, 2)
    assert np.all(np.diff(r[:, 0]) > 0) and np.all(r[:, 1] - r[:, 0] > thr)
    for acc in (False, True):
        y0 = rng.standard_normal(nrows)
        y0[::5] = -0.0
        yd = ds.DenseVector(torch.from_numpy(y0.copy()).to(DEV))
        (ds.spmv_add if acc else ds.spmv)(ds.SERIAL, a, ds.DenseVector(torch.from_numpy(x).to(DEV)), yd)
        torch.cuda.synchronize()
        want_y = want(nrows, ncols, rows, cols, vals, x, y0, acc)
        assert yd.data.cpu().numpy().tobytes() == want_y.tobytes(), acc


TILE_CASES = dict(CASES)
TILE_CASES["long_rows_and_gaps"] = lambda rng: (6000, 30000, np.concatenate([
    rng.integers(0, 40, 2000), np.zeros(1500, np.int64),                    # a long gap
    np.array([130, 511, 512, 513, 1500, 2049, 5000, 1, 0, 1]),              # chains, long runs
    rng.integers(5, 20, 2490)]))


@pytest.mark.parametrize("long_runs", [True, False])
@pytest.mark.parametrize("name", sorted(TILE_CASES))
def test_coo_descriptor_path_bitwise(name, long_runs, monkeypatch):
    """Row-sorted COO through the descriptor (ds_spmv: the pipeline for rows
    <= 27, else the warp-segment kernel, rows past the long-run threshold on
    the side kernel -- or, without that plan, in the warp kernel): absent
    rows, long gaps, rows around every tile size -- bitwise vs np.bincount."""
    import paper_2209_06478_b200 as ds
    from paper_2209_06478_b200 import kernels as K_
    if not long_runs:
        monkeypatch.setenv("DS_COO_NO_LONG_RUNS", "1")
    rng = np.random.default_rng(zlib.crc32(name.encode()) + 7)
    nrows, ncols, lengths = TILE_CASES[name](rng)
    rows, cols, vals = sorted_coo(rng, nrows, ncols, lengths)
    x = rng.standard_normal(ncols)
    a = ds.CooMatrix(nrows, ncols, rows, cols, vals, ds.MemorySpace.DEVICE, DEV)
    runs, cnt = K_.coo_long_runs(a)
    assert (cnt > 0) == (long_runs and lengths.max() > int(_native.load().ds_coo_long_run_threshold()))
    xt = ds.DenseVector(torch.from_numpy(x).to(DEV))
    for acc in (False, True):
        y0 = rng.standard_normal(nrows)
        y0[::7] = -0.0
        yd = ds.DenseVector(torch.from_numpy(y0.copy()).to(DEV))
        (ds.spmv_add if acc else ds.spmv)(ds.SERIAL, a, xt, yd)
        torch.cuda.synchronize()
        ref = want(nrows, ncols, rows, cols, vals, x, y0, acc)
        assert yd.data.cpu().numpy().tobytes() == ref.tobytes(), (name, acc)
