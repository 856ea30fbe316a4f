"""GPU parity: device kernels vs the reference's own outputs (golden fixtures
from tests/golden/make_golden.py) and vs the oracle.

Bar (BASELINE.md §4 / SURVEY §8c): conversions, index structures and
CSR / DIA / sorted-COO SpMV are BITWISE equal; unsorted COO within 1e-13
relative (the reference's threaded-COO tolerance, kernels.py:13-15); dot
within 1e-12 relative; CG iterations +-1 and residual history within 1e-8
relative.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import digest, golden_hashes, relative_error

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2209_06478_b200 as ds  # noqa: E402
from paper_2209_06478_b200 import kernels as K_  # noqa: E402
from oracle import dynsparse_oracle as O  # noqa: E402

DEV = torch.device("cuda", 0)
F = ds.FormatId


def dvec(a):
    return ds.DenseVector(torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(DEV))


def host(t):
    return t.detach().cpu().numpy()


def corpus(K):
    for case in range(int(K["ncase"][0])):
        key = f"c{case:03d}"
        nr, nc = (int(v) for v in K[f"{key}/dims"])
        yield key, nr, nc


def raw_device_coo(K, key, nr, nc):
    return ds.CooMatrix(nr, nc, K[f"{key}/in_rows"], K[f"{key}/in_cols"], K[f"{key}/in_vals"],
                        ds.MemorySpace.DEVICE, DEV)


def test_conversions_bitwise_from_raw_coo(K):
    for key, nr, nc in corpus(K):
        src = raw_device_coo(K, key, nr, nc)
        c = ds.convert(src, F.COO, fill_limit=2**62)
        assert np.array_equal(host(c.row_indices), K[f"{key}/coo/a0"]), key
        assert np.array_equal(host(c.col_indices), K[f"{key}/coo/a1"]), key
        assert host(c.values).tobytes() == K[f"{key}/coo/a2"].tobytes(), key
        s = ds.convert(src, F.CSR, fill_limit=2**62)
        assert np.array_equal(host(s.row_offsets), K[f"{key}/csr/a0"]), key
        assert np.array_equal(host(s.col_indices), K[f"{key}/csr/a1"]), key
        assert host(s.values).tobytes() == K[f"{key}/csr/a2"].tobytes(), key
        d = ds.convert(src, F.DIA, fill_limit=2**62)
        assert np.array_equal(host(d.offsets), K[f"{key}/dia/a0"]), key
        assert host(d.values).tobytes() == K[f"{key}/dia/a1"].tobytes(), key


def test_conversion_closure_every_pair(K):
    """src -> target -> source equals the canonical COO bitwise (test_datamove.py:167-177)."""
    for key, nr, nc in list(corpus(K))[:12]:
        ref = (K[f"{key}/coo/a0"], K[f"{key}/coo/a1"], K[f"{key}/coo/a2"])
        if not np.all(ref[2] != 0.0):
            continue  # explicit zeros are (correctly) dropped by DIA
        src = raw_device_coo(K, key, nr, nc)
        for sf in F:
            a = ds.convert(src, sf, fill_limit=2**62)
            for tf in F:
                back = ds.convert(ds.convert(a, tf, fill_limit=2**62), F.COO, fill_limit=2**62)
                assert np.array_equal(host(back.row_indices), ref[0])
                assert np.array_equal(host(back.col_indices), ref[1])
                assert host(back.values).tobytes() == ref[2].tobytes()


def test_fill_limit_iff_and_default(K):
    for key, nr, nc in corpus(K):
        src = raw_device_coo(K, key, nr, nc)
        slots, *dec = K[f"{key}/fill_decisions"].tolist()
        for lim, want in zip((slots - 1, slots, slots + 1), dec):
            if want:
                with pytest.raises(ds.DiaFillOverflow):
                    ds.convert(src, F.DIA, fill_limit=lim)
            else:
                ds.convert(src, F.DIA, fill_limit=lim)
        for fmt, want in zip(F, K[f"{key}/default_fill"].tolist()):
            mid = ds.convert(src, fmt, fill_limit=2**62)
            if want:
                with pytest.raises(ds.DiaFillOverflow):
                    ds.convert(mid, F.DIA)
            else:
                ds.convert(mid, F.DIA)


def _mats(K, key, nr, nc):
    return {
        "coo": ds.CooMatrix(nr, nc, K[f"{key}/coo/a0"], K[f"{key}/coo/a1"], K[f"{key}/coo/a2"],
                            ds.MemorySpace.DEVICE, DEV),
        "csr": ds.CsrMatrix(nr, nc, K[f"{key}/csr/a0"], K[f"{key}/csr/a1"], K[f"{key}/csr/a2"],
                            ds.MemorySpace.DEVICE, DEV),
        "dia": ds.DiaMatrix(nr, nc, K[f"{key}/dia/a0"], K[f"{key}/dia/a1"],
                            ds.MemorySpace.DEVICE, DEV),
    }


def test_spmv_and_spmv_add_bitwise(K):
    for key, nr, nc in corpus(K):
        x = dvec(K[f"{key}/x"])
        for name, m in _mats(K, key, nr, nc).items():
            for variant in (m, ds.DynamicMatrix(m)):
                y = ds.DenseVector.zeros(nr, ds.MemorySpace.DEVICE, DEV)
                y.data.fill_(123.0)  # spmv overwrites
                ds.spmv(ds.SERIAL, variant, x, y)
                assert host(y.data).tobytes() == K[f"{key}/{name}/spmv"].tobytes(), (key, name)
                ya = dvec(K[f"{key}/y0"])
                ds.spmv_add(ds.SERIAL, variant, x, ya)
                assert host(ya.data).tobytes() == K[f"{key}/{name}/spmv_add"].tobytes(), (key, name)


def test_raw_coo_spmv_tolerance(K):
    for key, nr, nc in corpus(K):
        src = raw_device_coo(K, key, nr, nc)
        y = ds.DenseVector.zeros(nr, ds.MemorySpace.DEVICE, DEV)
        ds.spmv(ds.SERIAL, src, dvec(K[f"{key}/x"]), y)
        assert relative_error(host(y.data), K[f"{key}/raw/spmv"]) < 1e-13


def test_host_containers_run_on_device(K):
    """Reference-style numpy containers: staged through the GPU, same bits."""
    key = "c001"
    nr, nc = (int(v) for v in K[f"{key}/dims"])
    a = ds.build_csr(nr, nc, K[f"{key}/csr/a0"], K[f"{key}/csr/a1"], K[f"{key}/csr/a2"])
    y = ds.DenseVector.zeros(nr)
    ds.spmv(ds.SERIAL, a, ds.DenseVector(K[f"{key}/x"]), y)
    assert isinstance(y.data, np.ndarray)
    assert y.data.tobytes() == K[f"{key}/csr/spmv"].tobytes()
    d = ds.convert(a, F.DIA, fill_limit=2**62)
    assert isinstance(d.values, np.ndarray)
    assert d.values.tobytes() == K[f"{key}/dia/a1"].tobytes()


def test_long_rows_pairwise_recursion(K):
    offs, cols, vals, x = K["long/offsets"], K["long/cols"], K["long/vals"], K["long/x"]
    a = ds.CsrMatrix(offs.size - 1, x.size, offs, cols, vals, ds.MemorySpace.DEVICE, DEV)
    lr, nl = K_.csr_plan(a)
    assert nl == int(np.sum(np.diff(offs) > 129))
    y = ds.DenseVector.zeros(a.nrows, ds.MemorySpace.DEVICE, DEV)
    ds.spmv(ds.SERIAL, a, dvec(x), y)                      # planned: CTA per long row
    assert host(y.data).tobytes() == K["long/spmv"].tobytes()
    # un-planned path: the 8-lane group walks the recursion itself
    from paper_2209_06478_b200 import _device, _native
    y2 = torch.zeros(a.nrows, dtype=torch.float64, device=DEV)
    xt = torch.from_numpy(x).to(DEV)
    _native.call("ds_spmv_csr", a.nrows, a.ncols, a.nnz, a.row_offsets.data_ptr(),
                 a.col_indices.data_ptr(), a.values.data_ptr(), None, 0,
                 xt.data_ptr(), y2.data_ptr(), 0, _device.stream(DEV))
    assert host(y2).tobytes() == K["long/spmv"].tobytes()


def test_signed_zeros(K):
    offs, cols, vals, x = K["zero/offsets"], K["zero/cols"], K["zero/vals"], K["zero/x"]
    a = ds.CsrMatrix(offs.size - 1, x.size, offs, cols, vals, ds.MemorySpace.DEVICE, DEV)
    for name in ("csr", "coo", "dia"):
        m = a if name == "csr" else ds.convert(a, F[name.upper()], fill_limit=2**62)
        y = ds.DenseVector.zeros(a.nrows, ds.MemorySpace.DEVICE, DEV)
        ds.spmv(ds.SERIAL, m, dvec(x), y)
        assert host(y.data).tobytes() == K[f"zero/{name}/spmv"].tobytes(), name
        ya = dvec(np.full(a.nrows, -0.0))
        ds.spmv_add(ds.SERIAL, m, dvec(x), ya)
        assert host(ya.data).tobytes() == K[f"zero/{name}/spmv_add"].tobytes(), name
    dz = ds.CooMatrix(2, 3, [0, 0, 0, 1, 1, 1, 1], [1, 1, 1, 2, 2, 0, 2],
                      [-0.0, -0.0, -0.0, 0.0, -0.0, -0.0, -0.0], ds.MemorySpace.DEVICE, DEV)
    cz = ds.convert(dz, F.COO)
    assert np.array_equal(host(cz.row_indices), K["zero/canon_rows"])
    assert np.array_equal(host(cz.col_indices), K["zero/canon_cols"])
    assert host(cz.values).tobytes() == K["zero/canon_vals"].tobytes()


def test_vector_kernels(K):
    for n in (0, 1, 2, 17, 1000, 4096, 20011):
        x, y = dvec(K[f"vec{n}/x"]), dvec(K[f"vec{n}/y"])
        w = ds.DenseVector.zeros(n, ds.MemorySpace.DEVICE, DEV)
        ds.waxpby(ds.SERIAL, 0.37, x, -1.9, y, w)
        assert host(w.data).tobytes() == K[f"vec{n}/waxpby"].tobytes()
        assert host(ds.scan(ds.SERIAL, x).data).tobytes() == K[f"vec{n}/scan"].tobytes()
        assert ds.reduce(ds.SERIAL, x) == K[f"vec{n}/reduce"][0]
        d = ds.dot(ds.SERIAL, x, y)
        ref = K[f"vec{n}/dot"][0]
        scale = float(np.abs(K[f"vec{n}/x"]) @ np.abs(K[f"vec{n}/y"])) if n else 1.0
        assert abs(d - ref) <= 1e-12 * scale
    # aliasing: p = r + 2 p (test_kernels.py:195-199)
    p, r = dvec([1.0, 2.0]), dvec([3.0, 4.0])
    ds.waxpby(ds.SERIAL, 1.0, r, 2.0, p, p)
    assert host(p.data).tolist() == [5.0, 8.0]


def test_diagonal_extract_and_update(K):
    rng = np.random.default_rng(14)
    for key, nr, nc in list(corpus(K))[:15]:
        for name, m in _mats(K, key, nr, nc).items():
            d = ds.extract_diagonal(m)
            assert host(d.data).tobytes() == K[f"{key}/{name}/diag"].tobytes(), (key, name)
    # tridiagonal update/extract round trip in every format (test_kernels.py:288-293)
    n = 20
    rows, cols = [], []
    for i in range(n):
        for j in (i - 1, i, i + 1):
            if 0 <= j < n:
                rows.append(i)
                cols.append(j)
    coo = ds.build_coo(n, n, rows, cols, np.where(np.array(rows) == np.array(cols), 2.0, -1.0),
                       space=ds.MemorySpace.DEVICE, device=DEV)
    dnew = rng.standard_normal(n)
    for fmt in F:
        m = ds.convert(coo, fmt, fill_limit=2**62)
        ds.update_diagonal(m, dvec(dnew))
        assert host(ds.extract_diagonal(m).data).tobytes() == dnew.tobytes()
    upper = ds.build_coo(2, 2, [0], [1], [1.0], space=ds.MemorySpace.DEVICE, device=DEV)
    with pytest.raises(ds.StructurallyAbsentDiagonal) as err:
        ds.update_diagonal(upper, dvec([1.0, 1.0]))
    assert err.value.index == 0
    dup = ds.build_coo(2, 2, [0, 0, 1], [0, 0, 1], [1.0, 2.0, 1.0],
                       space=ds.MemorySpace.DEVICE, device=DEV)
    ds.update_diagonal(dup, dvec([7.0, 8.0]))
    assert host(dup.values).tolist() == [7.0, 0.0, 8.0]


def test_stencil_distributed_spmv_bitwise(K):
    for si in range(int(K["nspecs"][0])):
        key = f"st{si}"
        spec = ds.GridSpec(*K[f"{key}/spec"].tolist())
        prob = ds.generate_problem(spec, space=ds.MemorySpace.DEVICE, device=DEV)
        splits = [ds.split_local_remote(prob, k) for k in range(prob.npartitions)]
        n = spec.local_points
        xs = []
        for k, part in enumerate(prob.partitions):
            x = np.zeros(part.a_full.ncols)
            x[:n] = K[f"{key}/p{k}/x_after"][:n]
            xs.append(dvec(x))
        ys = [ds.DenseVector.zeros(n, ds.MemorySpace.DEVICE, DEV) for _ in prob.partitions]
        ds.distributed_spmv(ds.SERIAL, prob, splits, xs, ys)
        for k in range(prob.npartitions):
            assert host(xs[k].data).tobytes() == K[f"{key}/p{k}/x_after"].tobytes()
            assert host(ys[k].data).tobytes() == K[f"{key}/p{k}/dist_y"].tobytes()


def _check_history(got, want, it_got, it_want):
    """Iterations +-1 (test_solver.py:121); history within 1e-8 relative, with
    an absolute floor of 64 eps: once ||r||/||b|| reaches the rounding floor
    (~1e-17) both sides hold rounding noise and no relative bar applies."""
    assert abs(it_got - it_want) <= 1
    k = min(len(got), len(want))
    g, w = np.asarray(got[:k]), np.asarray(want[:k])
    tol = 1e-8 * w + 64 * np.finfo(np.float64).eps
    assert np.all(np.abs(g - w) <= tol), np.max(np.abs(g - w) / np.maximum(w, 1e-300))


@pytest.mark.parametrize("use_graph", [False, True])
def test_cg_distributed_vs_reference(K, use_graph):
    for si in range(int(K["nspecs"][0])):
        key = f"st{si}"
        if f"{key}/cg_iters" not in K:
            continue
        spec = ds.GridSpec(*K[f"{key}/spec"].tolist())
        prob = ds.generate_problem(spec, space=ds.MemorySpace.DEVICE, device=DEV)
        splits = [ds.split_local_remote(prob, k) for k in range(prob.npartitions)]
        res = ds.cg(ds.SERIAL, ds.DistributedOperator(prob, splits),
                    [p.b for p in prob.partitions], tol=1e-9, max_iters=500, use_graph=use_graph)
        it, conv = K[f"{key}/cg_iters"].tolist()
        assert res.converged == bool(conv)
        _check_history(res.residual_history, K[f"{key}/cg_hist"], res.iterations, it)
        for k in range(prob.npartitions):
            assert np.max(np.abs(host(res.x[k].data) - K[f"{key}/p{k}/cg_x"])) < 1e-8
        rep = ds.validate_solver(ds.SERIAL, prob, splits)
        passed, converged, iters = K[f"{key}/validate"].tolist()
        assert rep.passed == bool(passed) and rep.converged == bool(converged)
        assert abs(rep.iterations - iters) <= 1


def test_cg_single_every_format_16cubed(K):
    part = ds.generate_problem(ds.GridSpec(16, 16, 16), space=ds.MemorySpace.DEVICE,
                               device=DEV).partitions[0]
    for name in ("coo", "csr", "dia"):
        a = ds.convert(part.a_full, F[name.upper()])
        res = ds.cg(ds.SERIAL, ds.DynamicMatrix(a), part.b, tol=1e-9, max_iters=500)
        it, conv = K[f"cg16/{name}/iters"].tolist()
        assert res.converged
        _check_history(res.residual_history, K[f"cg16/{name}/hist"], res.iterations, it)
        assert np.max(np.abs(host(res.x.data) - 1.0)) < 1e-6
        assert np.max(np.abs(host(res.x.data) - K[f"cg16/{name}/x"])) < 1e-8


def test_cg_edge_cases():
    idx = np.arange(3)
    a = ds.build_coo(3, 3, idx, idx, [1.0, 1.0, 1.0], space=ds.MemorySpace.DEVICE, device=DEV)
    res = ds.cg(ds.SERIAL, a, dvec([4.0, -2.0, 9.0]), tol=1e-12, max_iters=10)
    assert res.converged and res.iterations == 1
    assert np.allclose(host(res.x.data), [4.0, -2.0, 9.0], rtol=0, atol=1e-14)
    two = ds.build_coo(2, 2, [0, 1], [0, 1], [2.0, 2.0], space=ds.MemorySpace.DEVICE, device=DEV)
    res = ds.cg(ds.SERIAL, two, dvec([2.0, 2.0]), x0=dvec([1.0, 1.0]), tol=1e-12, max_iters=10)
    assert res.converged and res.iterations == 0 and res.residual_history.size == 1
    neg = ds.build_coo(2, 2, [0, 1], [0, 1], [-1.0, -2.0], space=ds.MemorySpace.DEVICE,
                       device=DEV)
    with pytest.raises(ds.BreakdownZeroCurvature):
        ds.cg(ds.SERIAL, neg, dvec([1.0, 1.0]))
    # host (numpy) inputs: reference-style call, result back on the host
    res = ds.cg(ds.SERIAL, ds.build_coo(2, 2, [0, 1], [0, 1], [2.0, 3.0]),
                ds.DenseVector([2.0, 3.0]), tol=1e-12, max_iters=10)
    assert isinstance(res.x.data, np.ndarray) and res.residual_history[0] == 1.0


@pytest.mark.slow
def test_104_cubed_golden_hashes():
    """BASELINE config 2 at full size: generator, conversions and all three
    SpMV formats match the reference's digests bitwise."""
    H = golden_hashes()
    part = ds.generate_problem(ds.GridSpec(104, 104, 104)).partitions[0]
    a_h = part.a_full
    assert digest(a_h.row_offsets, a_h.col_indices, a_h.values) == H["st104/csr"]
    assert digest(part.b.data) == H["st104/b"]
    A = ds.to_device(a_h, DEV)
    x = dvec(np.random.default_rng(0).standard_normal(A.nrows))
    y = ds.DenseVector.zeros(A.nrows, ds.MemorySpace.DEVICE, DEV)
    for name in ("csr", "coo", "dia"):
        m = ds.convert(A, F[name.upper()])
        if name == "coo":
            arrs = (m.row_indices, m.col_indices, m.values)
        elif name == "csr":
            arrs = (m.row_offsets, m.col_indices, m.values)
        else:
            arrs = (m.offsets, m.values)
        hs = [host(t).astype(np.int64) if t.dtype == torch.int32 else host(t) for t in arrs]
        assert digest(*hs) == H[f"st104/convert_{name}"], name
        ds.spmv(ds.SERIAL, m, x, y)
        assert digest(host(y.data)) == H[f"st104/spmv_{name}"], name
        if name == "dia":
            back = ds.convert(m, F.CSR)
            assert digest(host(back.row_offsets).astype(np.int64),
                          host(back.col_indices).astype(np.int64),
                          host(back.values)) == H["st104/dia_to_csr"]


@pytest.mark.slow
def test_powerlaw_golden_hashes():
    """BASELINE config 4: ~54.5M nnz irregular matrix; sort + duplicate sums
    on the device, SpMV CSR (long-row recursion) and COO bitwise."""
    H = golden_hashes()
    raw = O.powerlaw_coo()
    assert raw.rows.size == H["pl/raw_nnz"]
    coo = ds.CooMatrix(raw.nrows, raw.ncols, raw.rows, raw.cols, raw.vals,
                       ds.MemorySpace.DEVICE, DEV)
    del raw
    csr = ds.convert(coo, F.CSR)
    assert csr.nnz == H["pl/nnz"]
    assert digest(host(csr.row_offsets).astype(np.int64), host(csr.col_indices).astype(np.int64),
                  host(csr.values)) == H["pl/csr"]
    x = dvec(np.random.default_rng(1).standard_normal(csr.nrows))
    y = ds.DenseVector.zeros(csr.nrows, ds.MemorySpace.DEVICE, DEV)
    ds.spmv(ds.SERIAL, csr, x, y)
    assert digest(host(y.data)) == H["pl/spmv_csr"]
    c2 = ds.convert(csr, F.COO)
    assert digest(host(c2.row_indices).astype(np.int64), host(c2.col_indices).astype(np.int64),
                  host(c2.values)) == H["pl/convert_coo"]
    ds.spmv(ds.SERIAL, c2, x, y)
    assert digest(host(y.data)) == H["pl/spmv_coo"]
    with pytest.raises(ds.DiaFillOverflow):
        ds.convert(csr, F.DIA)


def test_device_generator_bitwise_equals_host():
    """On-device generate_problem (ds_stencil_*) == host generator == reference
    structure, for every partition of several decompositions."""
    for sp in [(1, 1, 1, 1, 1, 1), (3, 3, 3, 1, 1, 1), (4, 3, 2, 2, 1, 1), (4, 4, 4, 2, 2, 2),
               (5, 4, 3, 1, 3, 2), (7, 5, 6, 3, 2, 2), (16, 16, 16, 1, 1, 1)]:
        spec = ds.GridSpec(*sp)
        for r in range(spec.npartitions):
            h = ds.generate_partition(spec, r)
            d = ds.generate_partition(spec, r, space=ds.MemorySpace.DEVICE, device=DEV)
            assert d.a_full.space == ds.MemorySpace.DEVICE
            assert np.array_equal(host(d.a_full.row_offsets), h.a_full.row_offsets)
            assert np.array_equal(host(d.a_full.col_indices), h.a_full.col_indices)
            assert host(d.a_full.values).tobytes() == h.a_full.values.tobytes()
            assert host(d.b.data).tobytes() == h.b.data.tobytes()
            assert d.a_full.ncols == h.a_full.ncols
            assert d.halo.ghost_count == h.halo.ghost_count
            for e1, e2 in zip(d.halo.exchanges, h.halo.exchanges):
                assert e1.neighbor == e2.neighbor
                assert np.array_equal(e1.send_local_indices, e2.send_local_indices)
                assert np.array_equal(e1.recv_ghost_slots, e2.recv_ghost_slots)
            assert np.array_equal(d.local_to_global, h.local_to_global)
            assert np.array_equal(d.ghost_to_global, h.ghost_to_global)


def test_device_split_bitwise_equals_reference(K):
    for si in range(int(K["nspecs"][0])):
        key = f"st{si}"
        spec = ds.GridSpec(*K[f"{key}/spec"].tolist())
        prob = ds.generate_problem(spec, space=ds.MemorySpace.DEVICE, device=DEV)
        for k in range(prob.npartitions):
            sp = ds.split_local_remote(prob, k)
            loc, rem = sp.local.payload, sp.remote.payload
            pk = f"{key}/p{k}"
            assert np.array_equal(host(loc.row_offsets), K[f"{pk}/loc_offsets"])
            assert np.array_equal(host(loc.col_indices), K[f"{pk}/loc_cols"])
            assert host(loc.values).tobytes() == K[f"{pk}/loc_vals"].tobytes()
            assert np.array_equal(host(rem.row_offsets), K[f"{pk}/rem_offsets"])
            assert np.array_equal(host(rem.col_indices), K[f"{pk}/rem_cols"])
            assert host(rem.values).tobytes() == K[f"{pk}/rem_vals"].tobytes()
            assert rem.ncols == prob.partitions[k].halo.ghost_count
