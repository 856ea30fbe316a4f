"""GPU parity of every branch of the CSR SpMV launcher (ds_csr.cu) against
the oracle's np.add.reduceat restatement (kernels.py:102-119): bitwise.

Branches: the TMA pipeline's 27- and 33-wide register paths, its serial path
(rows of 34..129 entries when the longest row is unknown), "fat" tiles that
do not fit a stage (read from global memory), rows skipped for the long-row
kernels (> 129 entries), accumulate (spmv_add), empty rows and matrices whose
row count is not a multiple of the tile.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2209_06478_b200 as ds  # noqa: E402
from paper_2209_06478_b200 import _device, _native  # noqa: E402
from paper_2209_06478_b200 import kernels as K_  # noqa: E402
from oracle import dynsparse_oracle as O  # noqa: E402

DEV = torch.device("cuda", 0)


def random_csr(rng, nrows, ncols, lengths):
    offs = np.zeros(nrows + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lengths)
    cols = np.empty(offs[-1], dtype=np.int64)
    for i in range(nrows):
        L = int(lengths[i])
        cols[offs[i]:offs[i + 1]] = np.sort(rng.choice(ncols, size=L, replace=False))
    vals = rng.standard_normal(offs[-1])
    # signed zeros and exact cancellations exercise the -0.0 identity
    vals[rng.random(vals.size) < 0.02] = -0.0
    return offs, cols, vals


def oracle_y(offs, cols, vals, x, y0=None, accumulate=False):
    n = offs.size - 1
    m = O.csr(n, x.size, offs, cols, vals)
    y = np.zeros(n) if y0 is None else y0.copy()
    (O.spmv_add if accumulate else O.spmv)(m, x, y)
    return y


def run_abi(a, x, y0, accumulate, plan):
    """ds_spmv_csr through the C ABI; plan=False passes no long-row plan."""
    y = torch.from_numpy(y0.copy()).to(DEV)
    xt = torch.from_numpy(x).to(DEV)
    lr, nl = K_.csr_plan(a) if plan else (None, 0)
    _native.call("ds_spmv_csr", a.nrows, a.ncols, a.nnz, a.row_offsets.data_ptr(),
                 a.col_indices.data_ptr(), a.values.data_ptr(),
                 lr.data_ptr() if lr is not None else None, nl,
                 xt.data_ptr(), y.data_ptr(), int(accumulate), _device.stream(DEV))
    torch.cuda.synchronize()
    return y.cpu().numpy()


def device_csr(offs, cols, vals, ncols):
    return ds.CsrMatrix(offs.size - 1, ncols, offs, cols, vals, ds.MemorySpace.DEVICE, DEV)


@pytest.mark.parametrize("maxlen", [1, 8, 9, 17, 27, 28, 33])
def test_pipe_register_paths_bitwise(maxlen):
    rng = np.random.default_rng(100 + maxlen)
    n, nc = 5 * 256 + 37, 3000
    lengths = rng.integers(0, maxlen + 1, n)
    lengths[rng.integers(0, n, 5)] = maxlen
    lengths[:3] = 0
    offs, cols, vals = random_csr(rng, n, nc, lengths)
    x = rng.standard_normal(nc)
    a = device_csr(offs, cols, vals, nc)
    for acc in (False, True):
        y0 = rng.standard_normal(n)
        want = oracle_y(offs, cols, vals, x, y0, acc)
        # descriptor path (max_row_len known -> 27 / 33 register width)
        y = ds.DenseVector(torch.from_numpy(y0.copy()).to(DEV))
        (ds.spmv_add if acc else ds.spmv)(ds.SERIAL, a, ds.DenseVector(torch.from_numpy(x).to(DEV)), y)
        assert y.data.cpu().numpy().tobytes() == want.tobytes(), (maxlen, acc)
        # direct C ABI (max_row_len unknown -> 33 wide)
        assert run_abi(a, x, y0, acc, True).tobytes() == want.tobytes(), (maxlen, acc)
        # no plan: the paired 8-lane kernel
        assert run_abi(a, x, y0, acc, False).tobytes() == want.tobytes(), (maxlen, acc)


def test_pipe_serial_fat_and_long_rows():
    """Rows of 34..129 (serial path), tiles over the stage capacity (fat:
    global loads) and rows > 129 (skipped, computed by the long-row kernels)
    through ds_spmv_csr with a plan."""
    rng = np.random.default_rng(7)
    n, nc = 4 * 256 + 5, 20000
    lengths = rng.integers(20, 34, n)
    lengths[300:560] = rng.integers(34, 130, 260)    # serial rows, fat tiles
    lengths[700] = 1000                              # long rows (warp kernel)
    lengths[701] = 9000                              # (CTA kernel)
    offs, cols, vals = random_csr(rng, n, nc, lengths)
    x = rng.standard_normal(nc)
    a = device_csr(offs, cols, vals, nc)
    for acc in (False, True):
        y0 = rng.standard_normal(n)
        want = oracle_y(offs, cols, vals, x, y0, acc)
        assert run_abi(a, x, y0, acc, True).tobytes() == want.tobytes(), acc
        assert run_abi(a, x, y0, acc, False).tobytes() == want.tobytes(), acc
        # descriptor path: longest row > 33 -> length bins; rows <= 33 on the
        # pipeline, 34..129 on the binned kernel, > 129 on the long-row kernels
        assert K_.csr_bins(a) is not None
        y = ds.DenseVector(torch.from_numpy(y0.copy()).to(DEV))
        (ds.spmv_add if acc else ds.spmv)(ds.SERIAL, a, ds.DenseVector(torch.from_numpy(x).to(DEV)), y)
        assert y.data.cpu().numpy().tobytes() == want.tobytes(), ("binned", acc)


def test_pipe_stencil_and_cg_fused_dot():
    """The 27-point stencil (max row 27) through the CG engine, whose CSR
    SpMV fuses p.Ap: iterations and history equal the oracle's."""
    spec = ds.GridSpec(24, 20, 16)
    part = ds.generate_problem(spec).partitions[0]
    A = ds.to_device(part.a_full, DEV)
    assert K_.descriptor(A).max_row_len == 27
    ref = O.stencil_partition(24, 20, 16)
    x = np.random.default_rng(3).standard_normal(A.ncols)
    y = ds.DenseVector.zeros(A.nrows, ds.MemorySpace.DEVICE, DEV)
    ds.spmv(ds.SERIAL, A, ds.DenseVector(torch.from_numpy(x).to(DEV)), y)
    want = np.zeros(A.nrows)
    O.spmv(ref.a_full, x, want)
    assert y.data.cpu().numpy().tobytes() == want.tobytes()
    res = ds.cg(ds.SERIAL, A, ds.to_device(part.b, DEV), tol=1e-9, max_iters=500)
    oref = O.cg(ref.a_full, ref.b, tol=1e-9, max_iters=500)
    assert res.converged and abs(res.iterations - oref.iterations) <= 1
    k = min(res.iterations, oref.iterations) + 1
    h = np.asarray(res.residual_history[:k])
    assert np.all(np.abs(h - oref.history[:k]) <= 1e-8 * oref.history[:k] + 64 * np.finfo(float).eps)


@pytest.mark.parametrize("fmt", ["csr", "coo", "dia"])
def test_empty_matrix_spmv_and_add(fmt):
    """nnz == 0 (the remote part of a partition without ghosts): y = 0, and
    spmv_add turns -0.0 into +0.0 exactly like y += 0.0 (kernels.py:196-198)."""
    n, nc = 1000, 7
    offs = np.zeros(n + 1, dtype=np.int64)
    a = ds.convert(ds.CsrMatrix(n, nc, offs, np.zeros(0, np.int64), np.zeros(0), ds.MemorySpace.DEVICE,
                                DEV), ds.FormatId[fmt.upper()], fill_limit=2**40)
    x = ds.DenseVector(torch.ones(nc, dtype=torch.float64, device=DEV))
    y0 = np.random.default_rng(5).standard_normal(n)
    y0[::3] = -0.0
    for acc in (False, True):
        y = ds.DenseVector(torch.from_numpy(y0.copy()).to(DEV))
        (ds.spmv_add if acc else ds.spmv)(ds.SERIAL, a, x, y)
        want = y0 + 0.0 if acc else np.zeros(n)
        assert y.data.cpu().numpy().tobytes() == want.tobytes(), (fmt, acc)


@pytest.mark.parametrize("seed", [0, 1])
def test_tiles_irregular_bitwise(seed):
    """The entry-tile kernel of irregular matrices (csr_tile_kernel: products
    entry-parallel, one lane per row summing in np.add.reduceat order) with
    tiles of > 32 rows (runs of 1-entry rows), long runs of empty rows, every
    pairwise boundary (m = 7 / 8 / 15 / 16 / 128 addends), rows just past
    kLongRow (130..138: the first pairwise splits) and rows cut into
    pairwise-leaf tiles up to 15000 entries -- bitwise."""
    rng = np.random.default_rng(300 + seed)
    n, nc = 6000, 50000
    lengths = np.minimum(n, np.floor(6.0 * (1.0 - rng.random(n)) ** (-1 / 1.8))).astype(np.int64)
    lengths = np.minimum(lengths, 2000)
    lengths[100:900] = 1                               # ~380 rows per tile
    lengths[1000:3000:2] = 0                           # empty rows inside tiles
    lengths[3000:3100] = 0
    for i, L in enumerate([8, 9, 16, 17, 128, 129, 130, 131, 137, 138, 256, 257, 511, 512, 513,
                           1024, 1025, 0, 2]):
        lengths[4000 + 7 * i] = L
    lengths[5000] = 15000                              # ~150 pairwise leaves, 38 leaf tiles
    offs, cols, vals = random_csr(rng, n, nc, lengths)
    x = rng.standard_normal(nc)
    x[rng.random(nc) < 0.01] = -0.0
    a = device_csr(offs, cols, vals, nc)
    assert K_.csr_bins(a) is not None
    xt = ds.DenseVector(torch.from_numpy(x).to(DEV))
    for acc in (False, True):
        y0 = rng.standard_normal(n)
        y0[:50] = -0.0
        want = oracle_y(offs, cols, vals, x, y0, acc)
        y = ds.DenseVector(torch.from_numpy(y0.copy()).to(DEV))
        (ds.spmv_add if acc else ds.spmv)(ds.SERIAL, a, xt, y)
        assert y.data.cpu().numpy().tobytes() == want.tobytes(), ("tiles", acc)
