"""Generate golden fixtures by running the REAL reference (dev container only).

Usage (in the dev container, where /root/reference is mounted read-only):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py [--large]

Writes
  tests/golden/kat_small.npz      inputs + reference outputs for small cases
  tests/golden/golden_hashes.json sha256 digests of reference outputs at the
                                  BASELINE.json config sizes (104^3 stencil,
                                  power-law irregular matrix) -- with --large

Nothing on the GPU box reads /root/reference: the fixtures produced here are
committed and travel with the repo.  The oracle (oracle/dynsparse_oracle.py)
is pinned against them by tests/test_oracle_golden.py, and the GPU parity
tests compare device results against the same digests.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def random_coo_arrays(rng, max_dim):
    """Same recipe as the reference suite's random_coo (tests/conftest.py:62-72)."""
    nrows = int(rng.integers(1, max_dim + 1))
    ncols = int(rng.integers(1, max_dim + 1))
    density = float(rng.uniform(0.01, 0.5))
    k = int(round(density * nrows * ncols))
    return (nrows, ncols, rng.integers(0, nrows, size=k), rng.integers(0, ncols, size=k),
            rng.standard_normal(k))


def small(ds, out):
    F = ds.FormatId
    rng = np.random.default_rng(20240)
    ncase = 0
    # --- random corpus: conversions, spmv, spmv_add, fill-limit decisions
    for case in range(40):
        nr, nc, r, c, v = random_coo_arrays(rng, 64 if case % 4 else 128)
        if case % 7 == 3:           # explicit zeros and -0.0 to exercise DIA drop
            v[::5] = 0.0
            v[1::11] = -0.0
        coo = ds.build_coo(nr, nc, r, c, v)
        key = f"c{case:03d}"
        out[f"{key}/dims"] = np.array([nr, nc], np.int64)
        out[f"{key}/in_rows"], out[f"{key}/in_cols"], out[f"{key}/in_vals"] = (
            coo.row_indices, coo.col_indices, coo.values)
        x = rng.standard_normal(nc)
        y0 = rng.standard_normal(nr)
        out[f"{key}/x"], out[f"{key}/y0"] = x, y0
        for name, fmt in (("coo", F.COO), ("csr", F.CSR), ("dia", F.DIA)):
            m = ds.convert(coo, fmt, fill_limit=2**62)
            if fmt == F.COO:
                arrs = (m.row_indices, m.col_indices, m.values)
            elif fmt == F.CSR:
                arrs = (m.row_offsets, m.col_indices, m.values)
            else:
                arrs = (m.offsets, m.values)
            for i, a in enumerate(arrs):
                out[f"{key}/{name}/a{i}"] = a
            y = ds.DenseVector.zeros(nr)
            ds.spmv(ds.SERIAL, m, ds.DenseVector(x), y)
            out[f"{key}/{name}/spmv"] = y.data.copy()
            ya = ds.DenseVector(y0.copy())
            ds.spmv_add(ds.SERIAL, m, ds.DenseVector(x), ya)
            out[f"{key}/{name}/spmv_add"] = ya.data.copy()
        # raw (unsorted, duplicated) COO spmv: entry-order bincount
        y = ds.DenseVector.zeros(nr)
        ds.spmv(ds.SERIAL, coo, ds.DenseVector(x), y)
        out[f"{key}/raw/spmv"] = y.data.copy()
        # fill-limit iff around the exact slot count
        slots = len(set((coo.col_indices - coo.row_indices).tolist())) * nr
        dec = []
        for lim in (slots - 1, slots, slots + 1):
            try:
                ds.convert(coo, F.DIA, fill_limit=lim)
                dec.append(0)
            except ds.DiaFillOverflow:
                dec.append(1)
        out[f"{key}/fill_decisions"] = np.array([slots, *dec], np.int64)
        # default fill-limit decision from each source format
        dflt = []
        for fmt in (F.COO, F.CSR, F.DIA):
            src = ds.convert(coo, fmt, fill_limit=2**62)
            try:
                ds.convert(src, F.DIA)
                dflt.append(0)
            except ds.DiaFillOverflow:
                dflt.append(1)
        out[f"{key}/default_fill"] = np.array(dflt, np.int64)
        # diagonal extract on every format
        for name, fmt in (("coo", F.COO), ("csr", F.CSR), ("dia", F.DIA)):
            m = ds.convert(coo, fmt, fill_limit=2**62)
            out[f"{key}/{name}/diag"] = ds.extract_diagonal(m).data.copy()
        ncase += 1
    out["ncase"] = np.array([ncase])

    # --- long CSR rows (pairwise recursion > 128) and mixed lengths
    lr = np.random.default_rng(77)
    lengths = np.array([0, 1, 2, 7, 8, 9, 15, 16, 17, 120, 128, 129, 130, 131, 200, 257,
                        1000, 1031, 4099, 15000, 3, 0, 64], np.int64)
    nrl = lengths.size
    ncl = 20000
    offs = np.zeros(nrl + 1, np.int64)
    np.cumsum(lengths, out=offs[1:])
    cols = np.concatenate([np.sort(lr.choice(ncl, L, replace=False)) for L in lengths])
    vals = lr.standard_normal(cols.size) * 10.0 ** lr.integers(-6, 6, cols.size)
    xl = lr.standard_normal(ncl)
    a = ds.build_csr(nrl, ncl, offs, cols, vals)
    y = ds.DenseVector.zeros(nrl)
    ds.spmv(ds.SERIAL, a, ds.DenseVector(xl), y)
    out["long/offsets"], out["long/cols"], out["long/vals"], out["long/x"] = offs, cols, vals, xl
    out["long/spmv"] = y.data.copy()

    # --- signed zeros: rows of products that are -0.0 / +0.0 (reduceat keeps -0.0)
    zr = np.random.default_rng(99)
    zlen = np.array([1, 2, 3, 7, 8, 9, 10, 16, 17, 27, 0, 1, 2, 140, 5], np.int64)
    zoffs = np.zeros(zlen.size + 1, np.int64)
    np.cumsum(zlen, out=zoffs[1:])
    zcols = np.concatenate([np.sort(zr.choice(300, L, replace=False)) for L in zlen])
    zvals = zr.choice(np.array([0.0, -0.0, 1.0, -1.0]), zcols.size, p=[0.4, 0.4, 0.1, 0.1])
    zx = zr.choice(np.array([0.0, -0.0, 2.0, -3.0]), 300, p=[0.3, 0.3, 0.2, 0.2])
    az = ds.build_csr(zlen.size, 300, zoffs, zcols, zvals)
    out["zero/offsets"], out["zero/cols"], out["zero/vals"], out["zero/x"] = zoffs, zcols, zvals, zx
    for name, fmt in (("csr", F.CSR), ("coo", F.COO), ("dia", F.DIA)):
        m = az if fmt == F.CSR else ds.convert(az, fmt, fill_limit=2**62)
        y = ds.DenseVector.zeros(zlen.size)
        ds.spmv(ds.SERIAL, m, ds.DenseVector(zx), y)
        out[f"zero/{name}/spmv"] = y.data.copy()
        ya = ds.DenseVector(np.full(zlen.size, -0.0))
        ds.spmv_add(ds.SERIAL, m, ds.DenseVector(zx), ya)
        out[f"zero/{name}/spmv_add"] = ya.data.copy()
    # duplicates summed to signed zeros by canonicalisation
    dz = ds.build_coo(2, 3, [0, 0, 0, 1, 1, 1, 1], [1, 1, 1, 2, 2, 0, 2],
                      [-0.0, -0.0, -0.0, 0.0, -0.0, -0.0, -0.0])
    cz = ds.convert(dz, F.COO)
    out["zero/canon_rows"], out["zero/canon_cols"], out["zero/canon_vals"] = (
        cz.row_indices, cz.col_indices, cz.values)

    # --- dense-vector kernels
    vr = np.random.default_rng(13)
    for n in (0, 1, 2, 17, 1000, 4096, 20011):
        x = vr.standard_normal(n) * 10.0 ** vr.integers(-8, 8)
        yv = vr.standard_normal(n)
        w = ds.DenseVector.zeros(n)
        ds.waxpby(ds.SERIAL, 0.37, ds.DenseVector(x), -1.9, ds.DenseVector(yv), w)
        out[f"vec{n}/x"], out[f"vec{n}/y"] = x, yv
        out[f"vec{n}/waxpby"] = w.data.copy()
        out[f"vec{n}/scan"] = ds.scan(ds.SERIAL, ds.DenseVector(x)).data.copy()
        out[f"vec{n}/reduce"] = np.array([ds.reduce(ds.SERIAL, ds.DenseVector(x))])
        out[f"vec{n}/dot"] = np.array([ds.dot(ds.SERIAL, ds.DenseVector(x), ds.DenseVector(yv))])

    # --- stencil problems: structure, halo plans, splits, distributed spmv, cg
    specs = [(1, 1, 1, 1, 1, 1), (3, 3, 3, 1, 1, 1), (4, 3, 2, 2, 1, 1), (4, 4, 4, 2, 1, 1),
             (3, 2, 2, 2, 2, 1), (4, 4, 4, 2, 2, 2), (5, 4, 3, 1, 3, 2), (8, 8, 8, 1, 1, 2)]
    out["nspecs"] = np.array([len(specs)])
    for si, sp in enumerate(specs):
        spec = ds.GridSpec(*sp)
        prob = ds.generate_problem(spec)
        key = f"st{si}"
        out[f"{key}/spec"] = np.array(sp, np.int64)
        splits = [ds.split_local_remote(prob, k) for k in range(prob.npartitions)]
        gr = np.random.default_rng(21 + si)
        xs = []
        for k, part in enumerate(prob.partitions):
            pk = f"{key}/p{k}"
            a = part.a_full
            out[f"{pk}/offsets"], out[f"{pk}/cols"], out[f"{pk}/vals"] = (
                a.row_offsets, a.col_indices, a.values)
            out[f"{pk}/ncols"] = np.array([a.ncols])
            out[f"{pk}/b"] = part.b.data
            out[f"{pk}/l2g"], out[f"{pk}/g2g"] = part.local_to_global, part.ghost_to_global
            out[f"{pk}/nbrs"] = np.array([ex.neighbor for ex in part.halo.exchanges], np.int64)
            for ex in part.halo.exchanges:
                out[f"{pk}/send{ex.neighbor}"] = ex.send_local_indices
                out[f"{pk}/recv{ex.neighbor}"] = ex.recv_ghost_slots
            loc, rem = splits[k].local.payload, splits[k].remote.payload
            out[f"{pk}/loc_offsets"], out[f"{pk}/loc_cols"], out[f"{pk}/loc_vals"] = (
                loc.row_offsets, loc.col_indices, loc.values)
            out[f"{pk}/rem_offsets"], out[f"{pk}/rem_cols"], out[f"{pk}/rem_vals"] = (
                rem.row_offsets, rem.col_indices, rem.values)
            x = np.zeros(a.ncols)
            x[:a.nrows] = gr.standard_normal(a.nrows)
            xs.append(ds.DenseVector(x))
        ys = [ds.DenseVector.zeros(spec.local_points) for _ in prob.partitions]
        ds.distributed_spmv(ds.SERIAL, prob, splits, xs, ys)
        for k in range(prob.npartitions):
            out[f"{key}/p{k}/x_after"] = xs[k].data.copy()
            out[f"{key}/p{k}/dist_y"] = ys[k].data.copy()
        if spec.local_points <= 4096:
            op = ds.DistributedOperator(prob, splits)
            res = ds.cg(ds.SERIAL, op, [p.b for p in prob.partitions], tol=1e-9, max_iters=500)
            out[f"{key}/cg_iters"] = np.array([res.iterations, int(res.converged)])
            out[f"{key}/cg_hist"] = res.residual_history
            for k in range(prob.npartitions):
                out[f"{key}/p{k}/cg_x"] = res.x[k].data.copy()
            rep = ds.validate_solver(ds.SERIAL, prob, splits)
            out[f"{key}/validate"] = np.array([rep.passed, rep.converged, rep.iterations])
            out[f"{key}/validate_res"] = np.array([rep.final_residual])
    # single-matrix CG, 16^3 (config 1) in each format
    prob = ds.generate_problem(ds.GridSpec(16, 16, 16))
    part = prob.partitions[0]
    for name, fmt in (("coo", F.COO), ("csr", F.CSR), ("dia", F.DIA)):
        res = ds.cg(ds.SERIAL, ds.convert(part.a_full, fmt), part.b, tol=1e-9, max_iters=500)
        out[f"cg16/{name}/iters"] = np.array([res.iterations, int(res.converged)])
        out[f"cg16/{name}/hist"] = res.residual_history
        out[f"cg16/{name}/x"] = res.x.data.copy()


def large(ds, hashes):
    F = ds.FormatId
    t0 = time.time()
    prob = ds.generate_problem(ds.GridSpec(104, 104, 104))
    a = prob.partitions[0].a_full
    n = a.nrows
    hashes["st104/csr"] = digest(a.row_offsets, a.col_indices, a.values)
    hashes["st104/b"] = digest(prob.partitions[0].b.data)
    x = np.random.default_rng(0).standard_normal(n)
    for name, fmt in (("csr", F.CSR), ("coo", F.COO), ("dia", F.DIA)):
        m = ds.convert(a, fmt)
        if fmt == F.COO:
            hashes[f"st104/convert_{name}"] = digest(m.row_indices, m.col_indices, m.values)
        elif fmt == F.CSR:
            hashes[f"st104/convert_{name}"] = digest(m.row_offsets, m.col_indices, m.values)
        else:
            hashes[f"st104/convert_{name}"] = digest(m.offsets, m.values)
        y = ds.DenseVector.zeros(n)
        ds.spmv(ds.SERIAL, m, ds.DenseVector(x), y)
        hashes[f"st104/spmv_{name}"] = digest(y.data)
        if fmt == F.DIA:
            back = ds.convert(m, F.CSR)
            hashes["st104/dia_to_csr"] = digest(back.row_offsets, back.col_indices, back.values)
    print(f"104^3 done in {time.time() - t0:.1f}s", flush=True)
    # 104^3 x (2,2,2): partition 0 split sizes + remote arrays
    t0 = time.time()
    spec = ds.GridSpec(104, 104, 104, 2, 2, 2)
    # generate only what we need: the reference builds all 8 partitions
    prob = ds.generate_problem(spec)
    for k in (0, 7):
        part = prob.partitions[k]
        sp = ds.split_local_remote(prob, k)
        rem = sp.remote.payload
        hashes[f"st104x8/p{k}/a_full"] = digest(part.a_full.row_offsets, part.a_full.col_indices,
                                                part.a_full.values)
        hashes[f"st104x8/p{k}/remote"] = digest(rem.row_offsets, rem.col_indices, rem.values)
        hashes[f"st104x8/p{k}/ghosts"] = int(part.halo.ghost_count)
        hashes[f"st104x8/p{k}/nnz"] = int(part.a_full.nnz)
    print(f"104^3x8 done in {time.time() - t0:.1f}s", flush=True)
    # power-law irregular matrix
    t0 = time.time()
    rng = np.random.default_rng(2209)
    n = 4_194_304
    L = np.minimum(n, np.floor(6.0 * (1.0 - rng.random(n)) ** (-1 / 1.8))).astype(np.int64)
    rows = np.repeat(np.arange(n), L)
    cols = rng.integers(0, n, rows.size)
    vals = rng.standard_normal(rows.size)
    coo = ds.build_coo(n, n, rows, cols, vals)
    hashes["pl/raw_nnz"] = int(rows.size)
    csr = ds.convert(coo, F.CSR)
    hashes["pl/csr"] = digest(csr.row_offsets, csr.col_indices, csr.values)
    hashes["pl/nnz"] = int(csr.nnz)
    x = np.random.default_rng(1).standard_normal(n)
    y = ds.DenseVector.zeros(n)
    ds.spmv(ds.SERIAL, csr, ds.DenseVector(x), y)
    hashes["pl/spmv_csr"] = digest(y.data)
    ccoo = ds.convert(csr, F.COO)
    hashes["pl/convert_coo"] = digest(ccoo.row_indices, ccoo.col_indices, ccoo.values)
    y2 = ds.DenseVector.zeros(n)
    ds.spmv(ds.SERIAL, ccoo, ds.DenseVector(x), y2)
    hashes["pl/spmv_coo"] = digest(y2.data)
    try:
        ds.convert(csr, F.DIA)
        hashes["pl/dia_overflow"] = 0
    except ds.DiaFillOverflow as exc:
        hashes["pl/dia_overflow"] = 1
        hashes["pl/dia_overflow_msg"] = str(exc)
    print(f"power-law done in {time.time() - t0:.1f}s", flush=True)


def config_sizes(ds, hashes):
    """BASELINE config sizes the GPU parity tests pin (round 2):

    * config 3: the reference's CG at 104^3 (local DIA, tol 1e-9, the
      defaults): iteration count, the whole residual history and every
      997th entry of x -> cg104.npz (x itself is 9 MB);
    * config 5: the 192^3 partition's conversions (CSR->DIA, DIA->CSR,
      CSR->COO) and SpMV digests (DIA takes the x-window kernel on the GPU)."""
    t0 = time.time()
    F = ds.FormatId
    prob = ds.generate_problem(ds.GridSpec(104, 104, 104))
    part = prob.partitions[0]
    d = ds.convert(part.a_full, F.DIA)
    res = ds.cg(ds.ExecBackend.threaded(os.cpu_count() or 1), d, part.b, tol=1e-9, max_iters=500)
    x = np.asarray(res.x.data)
    np.savez_compressed(os.path.join(HERE, "cg104.npz"), history=np.asarray(res.residual_history),
                        iterations=res.iterations, converged=res.converged,
                        x_sample=x[::997].copy(), x_min=x.min(), x_max=x.max())
    hashes["cg104/iterations"] = int(res.iterations)
    print(f"cg104: {res.iterations} iterations in {time.time() - t0:.1f}s", flush=True)
    del prob, part, d, res
    # the reference's distributed CG at 16^3 per partition for the bench's
    # process grids of 2 / 4 / 8 GPUs (stencil.py:280-319, solver.py:120-189)
    dist = {}
    for procs in ((2, 1, 1), (2, 2, 1), (2, 2, 2)):
        prob = ds.generate_problem(ds.GridSpec(16, 16, 16, *procs))
        splits = [ds.split_local_remote(prob, k) for k in range(prob.npartitions)]
        res = ds.cg(ds.SERIAL, ds.DistributedOperator(prob, splits),
                    [p.b for p in prob.partitions], tol=1e-9, max_iters=500)
        key = "p%d%d%d" % procs
        dist[f"{key}/iterations"] = np.array(res.iterations)
        dist[f"{key}/history"] = np.asarray(res.residual_history)
        for k in range(prob.npartitions):
            dist[f"{key}/x{k}"] = np.asarray(res.x[k].data)
    np.savez_compressed(os.path.join(HERE, "cgdist16.npz"), **dist)
    print("cgdist16 done", flush=True)
    t0 = time.time()
    prob = ds.generate_problem(ds.GridSpec(192, 192, 192))
    a = prob.partitions[0].a_full
    hashes["st192/csr"] = digest(a.row_offsets, a.col_indices, a.values)
    n = a.nrows
    xv = np.random.default_rng(0).standard_normal(n)
    y = ds.DenseVector.zeros(n)
    ds.spmv(ds.SERIAL, a, ds.DenseVector(xv), y)
    hashes["st192/spmv_csr"] = digest(y.data)
    d = ds.convert(a, F.DIA)
    hashes["st192/convert_dia"] = digest(d.offsets, d.values)
    ds.spmv(ds.SERIAL, d, ds.DenseVector(xv), y)
    hashes["st192/spmv_dia"] = digest(y.data)
    back = ds.convert(d, F.CSR)
    hashes["st192/dia_to_csr"] = digest(back.row_offsets, back.col_indices, back.values)
    del back, d
    c = ds.convert(a, F.COO)
    hashes["st192/convert_coo"] = digest(c.row_indices, c.col_indices, c.values)
    print(f"192^3 done in {time.time() - t0:.1f}s", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--large", action="store_true")
    ap.add_argument("--config-sizes", action="store_true",
                    help="only add the config-3/5 keys (cg104.npz, st192/*) to golden_hashes.json")
    args = ap.parse_args()
    sys.path.insert(0, REF)
    import dynsparse as ds  # the real reference, read-only
    if args.config_sizes:
        path = os.path.join(HERE, "golden_hashes.json")
        with open(path) as fh:
            hashes = json.load(fh)
        config_sizes(ds, hashes)
        with open(path, "w") as fh:
            json.dump(hashes, fh, indent=1, sort_keys=True)
        return
    out: dict[str, np.ndarray] = {}
    small(ds, out)
    np.savez_compressed(os.path.join(HERE, "kat_small.npz"), **out)
    print(f"kat_small.npz: {len(out)} arrays")
    if args.large:
        hashes = {"numpy": np.__version__,
                  "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS")}
        large(ds, hashes)
        with open(os.path.join(HERE, "golden_hashes.json"), "w") as fh:
            json.dump(hashes, fh, indent=1, sort_keys=True)
        print(f"golden_hashes.json: {len(hashes)} entries")


if __name__ == "__main__":
    main()
