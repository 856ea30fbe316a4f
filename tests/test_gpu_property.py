"""Property-based GPU parity (hypothesis): random small COO matrices -- any
shape including empty, duplicates, explicit zeros and -0.0, unsorted entries
-- converted to every format on the device and multiplied, against the
oracle's restatement of the reference (datamove.py:208-295, kernels.py:102-198).

Bitwise: the converted index structures and values (one hop from COO, a
second hop from each result), the DIA fill-limit decision, CSR / DIA /
canonical-COO SpMV and spmv_add.  Each example is a few
kernel launches, so a hundred examples run in seconds.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
hypothesis = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

import paper_2209_06478_b200 as ds  # noqa: E402
from oracle import dynsparse_oracle as O  # noqa: E402

DEV = torch.device("cuda", 0)
FMT = {ds.FormatId.COO: O.COO, ds.FormatId.CSR: O.CSR, ds.FormatId.DIA: O.DIA}


@st.composite
def coo_inputs(draw):
    nrows = draw(st.integers(0, 40))
    ncols = draw(st.integers(0, 40))
    nnz = draw(st.integers(0, 160)) if nrows and ncols else 0
    seed = draw(st.integers(0, 2**31 - 1))
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, max(nrows, 1), nnz)
    cols = rng.integers(0, max(ncols, 1), nnz)
    if nnz and draw(st.booleans()):            # force duplicates
        k = rng.integers(0, nnz, nnz // 3 + 1)
        rows[k], cols[k] = rows[0], cols[0]
    vals = rng.standard_normal(nnz)
    mask = rng.random(nnz)
    vals[mask < 0.1] = 0.0
    vals[(mask >= 0.1) & (mask < 0.2)] = -0.0
    if nnz and draw(st.booleans()):            # exact cancellation inside a duplicate run
        vals[0] = 1.5
        vals[rng.integers(0, nnz)] = -1.5
    return nrows, ncols, rows, cols, vals, seed


def _host(m):
    """Device container -> the oracle's record (int64 indices, f64 values)."""
    if isinstance(m, ds.CooMatrix):
        return O.coo(m.nrows, m.ncols, m.row_indices.cpu().numpy(), m.col_indices.cpu().numpy(),
                     m.values.cpu().numpy())
    if isinstance(m, ds.CsrMatrix):
        return O.csr(m.nrows, m.ncols, m.row_offsets.cpu().numpy(), m.col_indices.cpu().numpy(),
                     m.values.cpu().numpy())
    return O.dia(m.nrows, m.ncols, m.offsets.cpu().numpy(), m.values.cpu().numpy())


def _same(a, b):
    if isinstance(a, O.OCoo):
        return (np.array_equal(a.rows, b.rows) and np.array_equal(a.cols, b.cols)
                and a.vals.tobytes() == b.vals.tobytes())
    if isinstance(a, O.OCsr):
        return (np.array_equal(a.offsets, b.offsets) and np.array_equal(a.cols, b.cols)
                and a.vals.tobytes() == b.vals.tobytes())
    return (np.array_equal(a.offsets, b.offsets) and a.values.shape == b.values.shape
            and a.values.tobytes() == b.values.tobytes())


@settings(max_examples=120, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(coo_inputs(), st.sampled_from([None, 0, 5, 40]))
def test_convert_and_spmv_match_oracle(inp, fill_limit):
    nrows, ncols, rows, cols, vals, seed = inp
    src = ds.CooMatrix(nrows, ncols, rows, cols, vals, ds.MemorySpace.DEVICE, DEV)
    osrc = O.coo(nrows, ncols, rows, cols, vals)
    rng = np.random.default_rng(seed + 1)
    x = rng.standard_normal(ncols)
    x[rng.random(ncols) < 0.1] = -0.0
    xt = ds.DenseVector(torch.from_numpy(x).to(DEV))
    for target in (ds.FormatId.COO, ds.FormatId.CSR, ds.FormatId.DIA):
        try:
            want = O.convert(osrc, FMT[target], fill_limit)
        except O.OracleFillOverflow:
            with pytest.raises(ds.DiaFillOverflow):
                ds.convert(src, target, fill_limit)
            continue
        got = ds.convert(src, target, fill_limit)
        assert _same(_host(got), want), (target, nrows, ncols, len(vals))
        # second hop from the device result (the canonical-CSR and DIA-source
        # fast paths): every target again, default fill limit
        for t2 in (ds.FormatId.COO, ds.FormatId.CSR, ds.FormatId.DIA):
            try:
                want2 = O.convert(want, FMT[t2])
            except O.OracleFillOverflow:
                with pytest.raises(ds.DiaFillOverflow):
                    ds.convert(got, t2)
                continue
            assert _same(_host(ds.convert(got, t2)), want2), (target, t2)
        # SpMV / spmv_add of the converted matrix: bitwise against the oracle
        # (COO: the canonical, row-sorted order -> np.bincount's sums)
        for acc in (False, True):
            y0 = rng.standard_normal(nrows)
            y0[::3] = -0.0
            yw = y0.copy()
            (O.spmv_add if acc else O.spmv)(want, x, yw)
            yd = ds.DenseVector(torch.from_numpy(y0.copy()).to(DEV))
            (ds.spmv_add if acc else ds.spmv)(ds.SERIAL, got, xt, yd)
            assert yd.data.cpu().numpy().tobytes() == yw.tobytes(), (target, acc)


@settings(max_examples=30, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(st.integers(2, 9), st.integers(2, 9), st.integers(2, 9), st.integers(1, 2),
       st.integers(1, 2), st.integers(1, 2),
       st.sampled_from(["coo", "csr", "dia"]), st.sampled_from(["coo", "csr"]),
       st.booleans())
def test_stencil_decompositions_match_oracle(nx, ny, nz, px, py, pz, lf, rf, use_graph):
    """Random 27-point decompositions generated on the device: each partition
    bitwise equal to the oracle's generator, the split's distributed SpMV
    bitwise against the oracle's in the same formats (local part COO / CSR /
    DIA, remote COO / CSR), and the distributed
    CG against the oracle's (iterations +-1, history within 1e-8, x within
    1e-8) -- the reference's stencil.py:143-319 and solver.py:120-189."""
    spec = ds.GridSpec(nx, ny, nz, px, py, pz)
    prob = ds.generate_problem(spec, space=ds.MemorySpace.DEVICE, device=DEV)
    oparts = O.stencil_problem(nx, ny, nz, px, py, pz)
    n = spec.local_points
    splits, osplits = [], []
    for k, (part, op) in enumerate(zip(prob.partitions, oparts)):
        a = _host(part.a_full)
        assert np.array_equal(a.offsets, op.a_full.offsets)
        assert np.array_equal(a.cols, op.a_full.cols)
        assert a.vals.tobytes() == op.a_full.vals.tobytes()
        sp = ds.split_local_remote(prob, k)
        if lf != "csr":
            ds.convert_inplace(sp.local, ds.FormatId[lf.upper()])
        if rf != "csr":
            ds.convert_inplace(sp.remote, ds.FormatId[rf.upper()])
        splits.append(sp)
        oloc, orem = O.split(op)
        # the oracle's parts in the same formats (the remote part of a
        # partition without ghosts is empty in any format)
        osplits.append((O.convert(oloc, FMT[ds.FormatId[lf.upper()]]),
                        O.convert(orem, FMT[ds.FormatId[rf.upper()]])))
    rng = np.random.default_rng(nx * 100 + ny * 10 + nz)
    xs_h = []
    for op in oparts:
        x = np.zeros(op.a_full.ncols)
        x[:n] = rng.standard_normal(n)
        xs_h.append(x)
    xs = [ds.DenseVector(torch.from_numpy(x.copy()).to(DEV)) for x in xs_h]
    ys = [ds.DenseVector.zeros(n, ds.MemorySpace.DEVICE, DEV) for _ in oparts]
    ds.distributed_spmv(ds.SERIAL, prob, splits, xs, ys)
    ys_h = [np.zeros(n) for _ in oparts]
    O.dist_spmv(oparts, osplits, xs_h, ys_h)
    for k in range(len(oparts)):
        assert xs[k].data.cpu().numpy().tobytes() == xs_h[k].tobytes()   # halo filled
        assert ys[k].data.cpu().numpy().tobytes() == ys_h[k].tobytes(), (k, lf, rf)
    res = ds.cg(ds.SERIAL, ds.DistributedOperator(prob, splits), [p.b for p in prob.partitions],
                tol=1e-9, max_iters=500, use_graph=use_graph)
    ref = O.cg_dist(oparts, osplits, [op.b for op in oparts], tol=1e-9, max_iters=500)
    assert abs(res.iterations - ref.iterations) <= 1 and res.converged == ref.converged
    k = min(res.iterations, ref.iterations) + 1
    h, w = np.asarray(res.residual_history[:k]), np.asarray(ref.history[:k])
    assert np.all(np.abs(h - w) <= 1e-8 * w + 64 * np.finfo(np.float64).eps)
    for kk in range(len(oparts)):
        assert np.max(np.abs(res.x[kk].data.cpu().numpy() - ref.x[kk])) < 1e-8


@settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(st.integers(1, 400), st.integers(1, 4000), st.integers(0, 2**31 - 1),
       st.sampled_from([34, 129, 130, 513, 3000]))
def test_irregular_csr_tiles_match_oracle(nrows, ncols, seed, longest):
    """Irregular CSR (longest row > 33: the row-tile / pairwise-leaf-tile
    grid, ds_csr_tiles) with random row lengths up to `longest` entries,
    empty rows, signed zeros: spmv and spmv_add bitwise vs np.add.reduceat's
    order (kernels.py:102-119); the COO form of the same matrix (warp
    segments + long-run kernel) bitwise vs np.bincount's."""
    rng = np.random.default_rng(seed)
    longest = min(longest, ncols)
    lengths = rng.integers(0, 12, nrows)
    lengths[rng.integers(0, nrows)] = longest
    lengths[rng.random(nrows) < 0.05] = 0
    lengths = np.minimum(lengths, ncols)
    offs = np.zeros(nrows + 1, dtype=np.int64)
    offs[1:] = np.cumsum(lengths)
    cols = np.concatenate([np.sort(rng.choice(ncols, size=int(L), replace=False))
                           for L in lengths]) if offs[-1] else np.zeros(0, np.int64)
    vals = rng.standard_normal(offs[-1])
    vals[rng.random(vals.size) < 0.03] = -0.0
    x = rng.standard_normal(ncols)
    x[rng.random(ncols) < 0.03] = -0.0
    a = ds.CsrMatrix(nrows, ncols, offs, cols, vals, ds.MemorySpace.DEVICE, DEV)
    oa = O.csr(nrows, ncols, offs, cols, vals)
    ac = ds.convert(a, ds.FormatId.COO)
    oc = O.convert(oa, O.COO)
    xt = ds.DenseVector(torch.from_numpy(x).to(DEV))
    for m, om in ((a, oa), (ac, oc)):
        for acc in (False, True):
            y0 = rng.standard_normal(nrows)
            y0[::4] = -0.0
            yw = y0.copy()
            (O.spmv_add if acc else O.spmv)(om, x, yw)
            yd = ds.DenseVector(torch.from_numpy(y0.copy()).to(DEV))
            (ds.spmv_add if acc else ds.spmv)(ds.SERIAL, m, xt, yd)
            assert yd.data.cpu().numpy().tobytes() == yw.tobytes(), (type(m).__name__, acc)


@settings(max_examples=15, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(st.integers(33_000, 90_000), st.integers(1, 9), st.integers(0, 3), st.integers(0, 2**31 - 1),
       st.sampled_from(["none", "dup", "swap"]))
def test_speculative_and_direct_paths_match_oracle(nrows, nd, extra, seed, damage):
    """Banded matrices large enough that the speculative DIA conversions
    sample (> 256 row tiles / 4096-entry chunks), plus `extra` entries on new
    diagonals in random rows (usually unsampled: a miss -> the census path)
    and optionally a duplicate or an unsorted pair (not canonical): CSR and
    COO sources to every target, bitwise against the oracle."""
    rng = np.random.default_rng(seed)
    ncols = nrows + int(rng.integers(-50, 50))
    band = np.sort(rng.choice(np.arange(-60, 61), size=nd, replace=False))
    rows = np.repeat(np.arange(nrows), nd)
    cols = rows + np.tile(band, nrows)
    for _ in range(extra):
        r = int(rng.integers(0, nrows))
        rows = np.append(rows, r)
        cols = np.append(cols, min(ncols - 1, r + int(rng.integers(100, 4000))))
    keep = (cols >= 0) & (cols < ncols)
    rows, cols = rows[keep], cols[keep]
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    uniq = np.ones(rows.size, bool)
    uniq[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
    rows, cols = rows[uniq], cols[uniq]
    vals = rng.standard_normal(rows.size)
    vals[rng.random(rows.size) < 0.05] = -0.0
    if damage != "none" and rows.size > 2:
        k = int(rng.integers(1, rows.size))
        while k < rows.size and rows[k] != rows[k - 1]:
            k += 1
        if k < rows.size:
            if damage == "dup":
                cols[k] = cols[k - 1]
            else:
                cols[k - 1], cols[k] = cols[k], cols[k - 1]
    offs = np.zeros(nrows + 1, np.int64)
    np.add.at(offs, rows + 1, 1)
    offs = np.cumsum(offs)
    srcs = ((ds.CsrMatrix(nrows, ncols, offs, cols, vals, ds.MemorySpace.DEVICE, DEV),
             O.csr(nrows, ncols, offs, cols, vals)),
            (ds.CooMatrix(nrows, ncols, rows, cols, vals, ds.MemorySpace.DEVICE, DEV),
             O.coo(nrows, ncols, rows, cols, vals)))
    for src, osrc in srcs:
        for target in (ds.FormatId.COO, ds.FormatId.CSR, ds.FormatId.DIA):
            want = O.convert(osrc, FMT[target])
            assert _same(_host(ds.convert(src, target)), want), (type(src).__name__, target,
                                                                   damage, extra)
