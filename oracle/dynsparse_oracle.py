"""CPU oracle for the dynsparse hot path  --  TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy restatement of the reference algorithm
(``/root/reference/pkg/src/dynsparse``) for exactly the functions on the hot
path: entry extraction, canonicalisation, COO/CSR/DIA conversion, SpMV per
format, the dense-vector kernels, the 27-point stencil generator with its
block decomposition and halo plan, the local/remote split, the halo gather,
distributed SpMV, CG and the diagonal-modification validation, and the tuner's
plan selection.  Every function cites the reference file:line it restates.

Who may use it: ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs -- as the *checker* or as the
timed CPU baseline.  The product package ``paper_2209_06478_b200`` never
imports it (a test enforces that), so there is no CPU fallback path.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference in the
dev container and commits fixtures/hashes under ``tests/golden``;
``tests/test_oracle_golden.py`` checks this oracle against them (and, when
``/root/reference`` is mounted, against the live reference on random inputs).

Arithmetic note: all floating-point reductions use the same numpy primitives
as the reference (``np.add.reduceat``, ``np.bincount``, ``np.cumsum``,
``np.dot``), so results are bitwise identical to the reference for the same
numpy build.  The integer work is exact by construction.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

COO, CSR, DIA = 0, 1, 2          # FormatId ABI, formats.py:33-42
FORMAT_NAMES = {COO: "coo", CSR: "csr", DIA: "dia"}

I64 = np.int64
F64 = np.float64


class OracleFillOverflow(Exception):
    """Mirror of DiaFillOverflow (errors.py:52-53)."""


class OracleBreakdown(Exception):
    """Mirror of BreakdownZeroCurvature (errors.py:81-82)."""


class OracleAbsentDiagonal(Exception):
    """Mirror of StructurallyAbsentDiagonal (errors.py:73-78)."""

    def __init__(self, index):
        super().__init__(index)
        self.index = index


# ---------------------------------------------------------------------------
# containers: plain records, int64 indices and float64 values (formats.py:82-87)
# ---------------------------------------------------------------------------

@dataclass
class OCoo:
    nrows: int
    ncols: int
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    fmt: int = COO


@dataclass
class OCsr:
    nrows: int
    ncols: int
    offsets: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    fmt: int = CSR


@dataclass
class ODia:
    nrows: int
    ncols: int
    offsets: np.ndarray
    values: np.ndarray        # C-contiguous (nrows, ndiags)
    fmt: int = DIA


def coo(nrows, ncols, rows, cols, vals) -> OCoo:
    return OCoo(int(nrows), int(ncols), np.ascontiguousarray(rows, I64),
                np.ascontiguousarray(cols, I64), np.ascontiguousarray(vals, F64))


def csr(nrows, ncols, offsets, cols, vals) -> OCsr:
    return OCsr(int(nrows), int(ncols), np.ascontiguousarray(offsets, I64),
                np.ascontiguousarray(cols, I64), np.ascontiguousarray(vals, F64))


def dia(nrows, ncols, offsets, values) -> ODia:
    return ODia(int(nrows), int(ncols), np.ascontiguousarray(offsets, I64),
                np.ascontiguousarray(values, F64))


def _dia_window(nrows: int, ncols: int, d: int) -> tuple[int, int]:
    """Rows i with 0 <= i + d < ncols, clipped to [0, nrows) (kernels.py:132-135)."""
    return max(0, -d), min(nrows, ncols - d)


def nnz(m) -> int:
    """Stored entries; DIA counts nonzero in-range slots (formats.py:166-167,205-206,239-255)."""
    if m.fmt == DIA:
        total = 0
        for j, d in enumerate(m.offsets.tolist()):
            lo, hi = _dia_window(m.nrows, m.ncols, d)
            if hi > lo:
                total += int(np.count_nonzero(m.values[lo:hi, j]))
        return total
    return int(m.vals.size)


# ---------------------------------------------------------------------------
# entry extraction and canonical COO (formats.py:439-479, datamove.py:208-235)
# ---------------------------------------------------------------------------

def entries(m):
    """(rows, cols, vals) of the stored entries, formats.py:439-479.

    CSR: row ids expanded from the offsets.  DIA: diagonal-major walk over
    the in-range window keeping only nonzero slots (explicit zeros and -0.0
    are dropped, formats.py:463-465)."""
    if m.fmt == COO:
        return m.rows, m.cols, m.vals
    if m.fmt == CSR:
        lengths = np.diff(m.offsets)
        return np.repeat(np.arange(m.nrows, dtype=I64), lengths), m.cols, m.vals
    r_out, c_out, v_out = [], [], []
    for j, d in enumerate(m.offsets.tolist()):
        lo, hi = _dia_window(m.nrows, m.ncols, d)
        if hi <= lo:
            continue
        column = m.values[lo:hi, j]
        keep = np.flatnonzero(column)
        if keep.size:
            r_out.append(keep + lo)
            c_out.append(keep + lo + d)
            v_out.append(column[keep])
    if not r_out:
        return np.zeros(0, I64), np.zeros(0, I64), np.zeros(0, F64)
    return np.concatenate(r_out), np.concatenate(c_out), np.concatenate(v_out)


def canonical(rows, cols, vals):
    """Stable (row, col) sort, duplicates summed as reduceat does (datamove.py:208-220).

    Duplicate runs are reduced with ``np.add.reduceat``: first element plus
    numpy's pairwise sum of the rest.  Zero sums are kept."""
    rows = np.asarray(rows, I64)
    cols = np.asarray(cols, I64)
    vals = np.asarray(vals, F64)
    if rows.size == 0:
        return rows.copy(), cols.copy(), vals.copy()
    perm = np.lexsort((cols, rows))
    rs, cs, vs = rows[perm], cols[perm], vals[perm]
    head = np.ones(rs.size, dtype=bool)
    head[1:] = (rs[1:] != rs[:-1]) | (cs[1:] != cs[:-1])
    starts = np.flatnonzero(head)
    return rs[starts], cs[starts], np.add.reduceat(vs, starts)


def canonical_coo(m) -> OCoo:
    """canonicalize_coo / _to_coo_proxy (datamove.py:223-235)."""
    r, c, v = canonical(*entries(m))
    return OCoo(m.nrows, m.ncols, r, c, v)


def default_fill_limit(m) -> int:
    """10 * max(nnz, nrows) of the SOURCE container (datamove.py:55-57)."""
    return 10 * max(nnz(m), m.nrows)


def canonical_to_csr(c: OCoo) -> OCsr:
    """Row histogram + inclusive scan into offsets[1:] (datamove.py:238-243)."""
    offsets = np.zeros(c.nrows + 1, I64)
    np.cumsum(np.bincount(c.rows, minlength=c.nrows), out=offsets[1:])
    return OCsr(c.nrows, c.ncols, offsets, c.cols, c.vals)


def canonical_to_dia(c: OCoo, fill_limit: int) -> ODia:
    """Distinct (col - row) diagonals, fill check before allocation, scatter
    (datamove.py:246-258)."""
    diag_of = c.cols - c.rows
    offs = np.unique(diag_of)
    slots = int(offs.size) * c.nrows
    if slots > fill_limit:
        raise OracleFillOverflow(f"{offs.size} diagonals x {c.nrows} rows > {fill_limit}")
    table = np.zeros((c.nrows, offs.size))
    if diag_of.size:
        table[c.rows, np.searchsorted(offs, diag_of)] = c.vals
    return ODia(c.nrows, c.ncols, offs, table)


def convert(m, target: int, fill_limit: int | None = None):
    """Every conversion goes src -> entries -> canonical COO -> target
    (datamove.py:261-281), including same-format rebuilds."""
    limit = default_fill_limit(m) if fill_limit is None else int(fill_limit)
    proxy = canonical_coo(m)
    if target == COO:
        return proxy
    if target == CSR:
        return canonical_to_csr(proxy)
    return canonical_to_dia(proxy, limit)


# ---------------------------------------------------------------------------
# SpMV (kernels.py:102-198) -- serial and row/entry-chunked threaded variants
# ---------------------------------------------------------------------------

_POOL: dict[int, ThreadPoolExecutor] = {}


def _pool(n: int) -> ThreadPoolExecutor:
    if n not in _POOL:
        _POOL[n] = ThreadPoolExecutor(max_workers=n)
    return _POOL[n]


def _spans(total: int, pieces: int):
    """Contiguous chunk bounds via linspace (kernels.py:74-75)."""
    edges = np.linspace(0, total, min(max(pieces, 1), max(total, 1)) + 1, dtype=I64)
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if a < b]


def _chunked(total: int, nthreads: int, body):
    spans = _spans(total, nthreads) if nthreads > 1 and total else [(0, total)]
    if len(spans) <= 1:
        body(0, total)
        return
    for fut in [_pool(nthreads).submit(body, a, b) for a, b in spans]:
        fut.result()


def spmv_csr(m: OCsr, x: np.ndarray, y: np.ndarray, nthreads: int = 1) -> None:
    """Per row: products, then np.add.reduceat over the row slice (kernels.py:102-119).
    Row sum order = p[first] + pairwise(p[first+1:end]); empty rows give 0."""
    off = m.offsets

    def block(r0, r1):
        e0, e1 = int(off[r0]), int(off[r1])
        y[r0:r1] = 0.0
        if e0 == e1:
            return
        prod = m.vals[e0:e1] * x[m.cols[e0:e1]]
        begins = off[r0:r1]
        filled = begins < off[r0 + 1:r1 + 1]
        y[r0:r1][filled] = np.add.reduceat(prod, (begins - e0)[filled])

    _chunked(m.nrows, nthreads, block)


def spmv_dia(m: ODia, x: np.ndarray, y: np.ndarray, nthreads: int = 1) -> None:
    """y = 0, then per diagonal ascending y[w] += values[w, j] * x[w + d]
    over the in-range window only (kernels.py:122-140)."""
    def block(r0, r1):
        y[r0:r1] = 0.0
        for j, d in enumerate(m.offsets.tolist()):
            lo = max(r0, -d, 0)
            hi = min(r1, m.nrows, m.ncols - d)
            if hi > lo:
                y[lo:hi] += m.values[lo:hi, j] * x[lo + d:hi + d]

    _chunked(m.nrows, nthreads, block)


def spmv_coo(m: OCoo, x: np.ndarray, y: np.ndarray, nthreads: int = 1) -> None:
    """bincount of products (sequential per row in entry order); threaded =
    per-chunk bincounts merged in chunk order (kernels.py:143-163)."""
    if nthreads <= 1 or m.rows.size == 0:
        y[:] = np.bincount(m.rows, weights=m.vals * x[m.cols], minlength=m.nrows)
        return
    spans = _spans(m.rows.size, nthreads)

    def part(span):
        a, b = span
        return np.bincount(m.rows[a:b], weights=m.vals[a:b] * x[m.cols[a:b]],
                           minlength=m.nrows)

    futs = [_pool(nthreads).submit(part, s) for s in spans]
    y[:] = 0.0
    for f in futs:
        y += f.result()


_SPMV = {COO: spmv_coo, CSR: spmv_csr, DIA: spmv_dia}


def spmv(m, x: np.ndarray, y: np.ndarray, nthreads: int = 1) -> None:
    """y = A x (overwrite), kernels.py:173-186."""
    assert x.size == m.ncols and y.size == m.nrows
    _SPMV[m.fmt](m, x, y, nthreads)


def spmv_add(m, x: np.ndarray, y: np.ndarray, nthreads: int = 1) -> None:
    """tmp = A x; y += tmp (kernels.py:189-198)."""
    tmp = np.zeros(m.nrows)
    _SPMV[m.fmt](m, x, tmp, nthreads)
    y += tmp


# ---------------------------------------------------------------------------
# dense-vector kernels (kernels.py:205-235)
# ---------------------------------------------------------------------------

def dot(x: np.ndarray, y: np.ndarray) -> float:
    """np.dot (OpenBLAS ddot; bits depend on OPENBLAS_NUM_THREADS), kernels.py:205-209."""
    return float(np.dot(x, y))


def waxpby(alpha: float, x: np.ndarray, beta: float, y: np.ndarray, w: np.ndarray) -> None:
    """w = alpha*x + beta*y, two rounded products then one rounded add (kernels.py:212-219)."""
    w[:] = alpha * x + beta * y


def reduce_sum(x: np.ndarray) -> float:
    """Sequential prefix order, last element (kernels.py:222-230)."""
    return 0.0 if x.size == 0 else float(np.cumsum(x)[-1])


def scan_sum(x: np.ndarray) -> np.ndarray:
    """Inclusive sequential prefix sums (kernels.py:233-235)."""
    return np.cumsum(x)


# ---------------------------------------------------------------------------
# diagonal extract / update (kernels.py:242-337)
# ---------------------------------------------------------------------------

def extract_diag(m) -> np.ndarray:
    n = min(m.nrows, m.ncols)
    if m.fmt == COO:
        on = m.rows == m.cols
        return np.bincount(m.rows[on], weights=m.vals[on], minlength=n)[:n]
    if m.fmt == CSR:
        out = np.zeros(n)
        r = np.repeat(np.arange(m.nrows, dtype=I64), np.diff(m.offsets))
        on = r == m.cols
        out[r[on]] = m.vals[on]
        return out
    where = np.flatnonzero(m.offsets == 0)
    if where.size == 0:
        return np.zeros(n)
    return m.values[:n, int(where[0])].copy()


def update_diag(m, d: np.ndarray) -> None:
    """In-place overwrite of A(i,i); COO duplicates: first stored occurrence
    takes the value, later ones become 0.0 (kernels.py:285-337)."""
    n = d.size
    if n == 0:
        return
    if m.fmt == DIA:
        where = np.flatnonzero(m.offsets == 0)
        if where.size == 0:
            raise OracleAbsentDiagonal(0)
        m.values[:n, int(where[0])] = d
        return
    if m.fmt == COO:
        pos = np.flatnonzero(m.rows == m.cols)
        hit = m.rows[pos]
    else:
        r = np.repeat(np.arange(m.nrows, dtype=I64), np.diff(m.offsets))
        pos = np.flatnonzero(r == m.cols)
        hit = r[pos]
    seen = np.zeros(n, dtype=bool)
    seen[hit] = True
    if not seen.all():
        raise OracleAbsentDiagonal(int(np.flatnonzero(~seen)[0]))
    if m.fmt == COO:
        m.vals[pos] = 0.0
        uniq, first = np.unique(hit, return_index=True)
        m.vals[pos[first]] = d[uniq]
    else:
        m.vals[pos] = d[hit]


# ---------------------------------------------------------------------------
# 27-point stencil problem with block decomposition (stencil.py:143-277)
# ---------------------------------------------------------------------------

DIAG_COEFF = 26.0          # stencil.py:29
OFF_COEFF = -1.0           # stencil.py:30


@dataclass
class OPart:
    rank: int
    coords: tuple
    a_full: OCsr
    b: np.ndarray
    ghost_count: int
    # list of (neighbor, send_local_indices, recv_ghost_slots), neighbors ascending
    exchanges: list = field(default_factory=list)
    local_to_global: np.ndarray | None = None
    ghost_to_global: np.ndarray | None = None


def stencil_partition(nx, ny, nz, px=1, py=1, pz=1, rank=0) -> OPart:
    """One partition of generate_problem (stencil.py:143-253).

    Local numbering x fastest; rank = cx + px*(cy + py*cz); neighbor order
    dz, dy, dx in (-1, 0, 1) with dx fastest; ghosts sorted by
    (owner rank, owner-local index); rows lexsorted by (row, col)."""
    n = nx * ny * nz
    gnx, gny, gnz = nx * px, ny * py, nz * pz
    cx, cy, cz = rank % px, (rank // px) % py, rank // (px * py)
    ids = np.arange(n, dtype=I64)
    gx = ids % nx + cx * nx
    gy = (ids // nx) % ny + cy * ny
    gz = ids // (nx * ny) + cz * nz
    row_l, own_l, loc_l, val_l = [], [], [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                tx, ty, tz = gx + dx, gy + dy, gz + dz
                ok = (tx >= 0) & (tx < gnx) & (ty >= 0) & (ty < gny) & (tz >= 0) & (tz < gnz)
                if not ok.any():
                    continue
                tx, ty, tz = tx[ok], ty[ok], tz[ok]
                ox, oy, oz = tx // nx, ty // ny, tz // nz
                row_l.append(ids[ok])
                own_l.append(ox + px * (oy + py * oz))
                loc_l.append((tx - ox * nx) + nx * ((ty - oy * ny) + ny * (tz - oz * nz)))
                c = DIAG_COEFF if dx == 0 and dy == 0 and dz == 0 else OFF_COEFF
                val_l.append(np.full(int(ok.sum()), c))
    rows = np.concatenate(row_l)
    owner = np.concatenate(own_l)
    oloc = np.concatenate(loc_l)
    vals = np.concatenate(val_l)
    far = owner != rank
    keys = np.unique(owner[far] * n + oloc[far])
    cols = np.where(far, 0, oloc).astype(I64)
    if keys.size:
        cols[far] = n + np.searchsorted(keys, owner[far] * n + oloc[far])
    perm = np.lexsort((cols, rows))
    rows, cols, vals = rows[perm], cols[perm], vals[perm]
    offsets = np.zeros(n + 1, I64)
    np.cumsum(np.bincount(rows, minlength=n), out=offsets[1:])
    b = np.bincount(rows, weights=vals, minlength=n)
    g_owner, g_local = keys // n, keys % n
    exchanges = []
    for q in np.unique(g_owner).tolist():
        sel = np.flatnonzero(g_owner == q)
        exchanges.append((int(q), g_local[sel].copy(), n + sel))
    l2g = gx + gnx * (gy + gny * gz)
    qx, qy, qz = g_owner % px, (g_owner // px) % py, g_owner // (px * py)
    g2g = ((g_local % nx + qx * nx) + gnx * (((g_local // nx) % ny + qy * ny)
                                          + gny * (g_local // (nx * ny) + qz * nz)))
    return OPart(rank, (cx, cy, cz), OCsr(n, n + int(keys.size), offsets, cols, vals),
                 b, int(keys.size), exchanges, l2g, g2g)


def stencil_problem(nx, ny, nz, px=1, py=1, pz=1) -> list[OPart]:
    return [stencil_partition(nx, ny, nz, px, py, pz, r) for r in range(px * py * pz)]


def split(part: OPart):
    """Local (cols < n, square) and remote (cols >= n shifted by -n) CSR parts
    (stencil.py:256-277)."""
    a = part.a_full
    n = a.nrows
    r = np.repeat(np.arange(n, dtype=I64), np.diff(a.offsets))
    inner = a.cols < n

    def side(mask, ncols, shift):
        off = np.zeros(n + 1, I64)
        np.cumsum(np.bincount(r[mask], minlength=n), out=off[1:])
        return OCsr(n, ncols, off, a.cols[mask] - shift, a.vals[mask])

    return side(inner, n, 0), side(~inner, part.ghost_count, n)


def exchange(parts: list[OPart], xs: list[np.ndarray]) -> None:
    """Ghost gather x_k[recv] = x_q[send] (stencil.py:280-295)."""
    for part, x in zip(parts, xs):
        for q, send, recv in part.exchanges:
            x[recv] = xs[q][send]


def dist_spmv(parts, splits, xs, ys, nthreads=1) -> None:
    """exchange; y = local x_owned; y += remote x_ghost (stencil.py:298-319)."""
    exchange(parts, xs)
    for k, (loc, rem) in enumerate(splits):
        n = loc.nrows
        spmv(loc, xs[k][:n], ys[k], nthreads)
        spmv_add(rem, xs[k][n:], ys[k], nthreads)


# ---------------------------------------------------------------------------
# conjugate gradient (solver.py:56-234)
# ---------------------------------------------------------------------------

@dataclass
class OCgResult:
    x: object
    iterations: int
    history: np.ndarray
    converged: bool


def cg(m, b: np.ndarray, x0=None, tol=1e-9, max_iters=500, nthreads=1) -> OCgResult:
    """Unpreconditioned CG on one matrix (solver.py:73-117)."""
    n = m.nrows
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=F64, copy=True)
    r, p, ap = np.zeros(n), np.zeros(n), np.zeros(n)
    spmv(m, x, ap, nthreads)
    waxpby(1.0, b, -1.0, ap, r)
    nb = math.sqrt(dot(b, b))
    scale = nb if nb > 0.0 else 1.0
    rr = dot(r, r)
    hist = [math.sqrt(rr) / scale]
    if hist[0] <= tol:
        return OCgResult(x, 0, np.asarray(hist), True)
    waxpby(1.0, r, 0.0, r, p)
    it, done = 0, False
    for k in range(1, max_iters + 1):
        it = k
        spmv(m, p, ap, nthreads)
        pap = dot(p, ap)
        if pap <= 0.0:
            raise OracleBreakdown(f"p'Ap = {pap} at iteration {k}")
        alpha = rr / pap
        waxpby(1.0, x, alpha, p, x)
        waxpby(1.0, r, -alpha, ap, r)
        rr_new = dot(r, r)
        hist.append(math.sqrt(rr_new) / scale)
        if hist[-1] <= tol:
            done = True
            break
        waxpby(1.0, r, rr_new / rr, p, p)
        rr = rr_new
    return OCgResult(x, it, np.asarray(hist), done)


def cg_dist(parts, splits, bs, x0s=None, tol=1e-9, max_iters=500, nthreads=1) -> OCgResult:
    """Distributed CG: rank-ordered sum of partition dots, p carries ghost
    slots sharing its owned prefix (solver.py:120-189)."""
    P = len(parts)
    n = parts[0].a_full.nrows

    def gdot(u, v):
        return sum(dot(u[k], v[k]) for k in range(P))

    x = [np.zeros(n) if x0s is None else np.array(x0s[k], dtype=F64, copy=True) for k in range(P)]
    p_full = [np.zeros(n + parts[k].ghost_count) for k in range(P)]
    p = [pf[:n] for pf in p_full]
    r = [np.zeros(n) for _ in range(P)]
    ap = [np.zeros(n) for _ in range(P)]
    for k in range(P):
        p[k][:] = x[k]
    dist_spmv(parts, splits, p_full, ap, nthreads)
    for k in range(P):
        waxpby(1.0, bs[k], -1.0, ap[k], r[k])
    nb = math.sqrt(gdot(bs, bs))
    scale = nb if nb > 0.0 else 1.0
    rr = gdot(r, r)
    hist = [math.sqrt(rr) / scale]
    if hist[0] <= tol:
        return OCgResult(x, 0, np.asarray(hist), True)
    for k in range(P):
        waxpby(1.0, r[k], 0.0, r[k], p[k])
    it, done = 0, False
    for i in range(1, max_iters + 1):
        it = i
        dist_spmv(parts, splits, p_full, ap, nthreads)
        pap = gdot(p, ap)
        if pap <= 0.0:
            raise OracleBreakdown(f"p'Ap = {pap} at iteration {i}")
        alpha = rr / pap
        for k in range(P):
            waxpby(1.0, x[k], alpha, p[k], x[k])
            waxpby(1.0, r[k], -alpha, ap[k], r[k])
        rr_new = gdot(r, r)
        hist.append(math.sqrt(rr_new) / scale)
        if hist[-1] <= tol:
            done = True
            break
        beta = rr_new / rr
        for k in range(P):
            waxpby(1.0, r[k], beta, p[k], p[k])
        rr = rr_new
    return OCgResult(x, it, np.asarray(hist), done)


def validate(parts, splits, diag_value=1.0e6, tol=1e-12, max_iters=50, bound=12):
    """Diagonal-modification check (solver.py:192-234); returns
    (passed, converged, iterations, final_residual); diagonals restored."""
    n = parts[0].a_full.nrows
    saved = [extract_diag(loc) for loc, _ in splits]
    try:
        for loc, _ in splits:
            update_diag(loc, np.full(n, diag_value))
        ones = [np.ones(n + p.ghost_count) for p in parts]
        bs = [np.zeros(n) for _ in parts]
        dist_spmv(parts, splits, ones, bs)
        res = cg_dist(parts, splits, bs, tol=tol, max_iters=max_iters)
    finally:
        for (loc, _), d in zip(splits, saved):
            update_diag(loc, d)
    passed = res.converged and res.iterations <= bound
    return passed, res.converged, res.iterations, float(res.history[-1])


# ---------------------------------------------------------------------------
# tuner plan selection (tuner.py:123-180)
# ---------------------------------------------------------------------------

def select_plan(entries: dict, nparts: int, mode: str):
    """entries: {(k, local_fmt, remote_fmt): seconds}.  Returns a list of
    (local, remote) per partition; ties go to the lower format id."""
    fmts = (COO, CSR, DIA)
    if mode == "fixed":
        return [(CSR, CSR)] * nparts
    if mode in ("morpheus", "ghost"):
        best = None
        for f in fmts:
            cells = [(k, f, CSR) if mode == "morpheus" else (k, CSR, f) for k in range(nparts)]
            if all(c in entries for c in cells):
                worst = max(entries[c] for c in cells)
                if best is None or worst < best[0]:
                    best = (worst, f)
        if best is None:
            raise ValueError("empty search space")
        pick = best[1]
        return [(pick, CSR) if mode == "morpheus" else (CSR, pick)] * nparts
    out = []
    for k in range(nparts):
        cands = [(entries[(k, a, b)], a, b) for a in fmts for b in fmts if (k, a, b) in entries]
        if not cands:
            raise ValueError(f"partition {k} has no measured combination")
        _, a, b = min(cands)
        out.append((a, b))
    return out


# ---------------------------------------------------------------------------
# synthetic irregular matrix of BASELINE.md (power-law row lengths)
# ---------------------------------------------------------------------------

def powerlaw_coo(n: int = 4_194_304, seed: int = 2209, shape: float = 1.8, xmin: float = 6.0) -> OCoo:
    """BASELINE.md §2 generator: L = min(n, floor(xmin (1-U)^(-1/shape)))."""
    rng = np.random.default_rng(seed)
    lengths = np.minimum(n, np.floor(xmin * (1.0 - rng.random(n)) ** (-1 / shape))).astype(I64)
    rows = np.repeat(np.arange(n, dtype=I64), lengths)
    cols = rng.integers(0, n, rows.size)
    vals = rng.standard_normal(rows.size)
    return OCoo(n, n, rows, cols.astype(I64), vals)


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# HPCG SymGS / MG -- NOT in the reference (SPEC.md:16,
# PAPER.md:166): PARITY UNPINNED against the reference.  This restates the
# HPCG benchmark's ComputeSYMGS_ref / ComputeMG_ref with the 8-colour
# ordering of the 27-point stencil (colour = x%2 + 2(y%2) + 4(z%2), local
# coordinates), under which rows of one colour are independent.  The device
# kernels are held to bitwise parity with these functions.
# ---------------------------------------------------------------------------

def stencil_colors(nx, ny, nz) -> np.ndarray:
    i = np.arange(nx * ny * nz, dtype=I64)
    return (i % nx) % 2 + 2 * (((i // nx) % ny) % 2) + 4 * ((i // (nx * ny)) % 2)


def symgs_colored(m: OCsr, r: np.ndarray, x: np.ndarray, colors: np.ndarray) -> None:
    """One symmetric Gauss-Seidel sweep in place: colours 0..7 forward, then
    7..0 backward.  Per row i: s = r[i]; s = s - a_ij * x[j] for every j != i
    in stored (ascending) column order; x[i] = s / a_ii (ComputeSYMGS_ref)."""
    off, cols, vals = m.offsets, m.cols, m.vals
    n = m.nrows
    order = [np.flatnonzero(colors == c) for c in range(8)]

    def relax(rows):
        for i in rows.tolist():
            s = r[i]
            d = 0.0
            for k in range(int(off[i]), int(off[i + 1])):
                j = int(cols[k])
                if j == i:
                    d = vals[k]
                else:
                    s = s - vals[k] * x[j]
            x[i] = s / d
    for c in range(8):
        relax(order[c])
    for c in range(7, -1, -1):
        relax(order[c])
    assert x.size == n


def mg_levels(nx, ny, nz, levels=4, fmt=CSR):
    """[(matrix, colors, f2c, op)] finest first; coarse grids halve every
    dimension while it stays even (GenerateCoarseProblem).  ``op`` is the
    level matrix converted to ``fmt`` -- the format the residual SpMVs run
    in (the smoother always walks the CSR rows)."""
    out = []
    for lev in range(levels):
        part = stencil_partition(nx, ny, nz)
        f2c = None
        if lev + 1 < levels and nx % 2 == 0 and ny % 2 == 0 and nz % 2 == 0:
            cx, cy, cz = nx // 2, ny // 2, nz // 2
            ic = np.arange(cx * cy * cz, dtype=I64)
            xc, yc, zc = ic % cx, (ic // cx) % cy, ic // (cx * cy)
            f2c = 2 * xc + nx * (2 * yc + ny * 2 * zc)
        a = part.a_full
        out.append((a, stencil_colors(nx, ny, nz), f2c, a if fmt == CSR else convert(a, fmt)))
        if f2c is None:
            break
        nx, ny, nz = nx // 2, ny // 2, nz // 2
    return out


def mg_vcycle(levels, lev: int, r: np.ndarray, x: np.ndarray) -> None:
    """ComputeMG_ref: x = 0; pre-smooth; Axf = A x; rc = r[f2c] - Axf[f2c];
    recurse; x[f2c] += xc; post-smooth (coarsest: one smooth)."""
    a, colors, f2c, op = levels[lev]
    x[:] = 0.0
    symgs_colored(a, r, x, colors)
    if f2c is None or lev + 1 >= len(levels):
        return
    axf = np.zeros(a.nrows)
    spmv(op, x, axf)
    rc = r[f2c] - axf[f2c]
    xc = np.zeros(f2c.size)
    mg_vcycle(levels, lev + 1, rc, xc)
    x[f2c] += xc
    symgs_colored(a, r, x, colors)


def pcg_mg(levels, b: np.ndarray, tol=1e-9, max_iters=50) -> OCgResult:
    """HPCG's preconditioned CG (ComputeCG_ref) with the MG preconditioner;
    history = ||r|| / ||b|| like the unpreconditioned solver."""
    a = levels[0][3]
    n = a.nrows
    x, r, z, p, ap = (np.zeros(n) for _ in range(5))
    spmv(a, x, ap)
    waxpby(1.0, b, -1.0, ap, r)
    nb = math.sqrt(dot(b, b))
    scale = nb if nb > 0.0 else 1.0
    hist = [math.sqrt(dot(r, r)) / scale]
    if hist[0] <= tol:
        return OCgResult(x, 0, np.asarray(hist), True)
    mg_vcycle(levels, 0, r, z)
    waxpby(1.0, z, 0.0, z, p)
    rtz = dot(r, z)
    it, done = 0, False
    for k in range(1, max_iters + 1):
        it = k
        spmv(a, p, ap)
        pap = dot(p, ap)
        if pap <= 0.0:
            raise OracleBreakdown(f"p'Ap = {pap} at iteration {k}")
        alpha = rtz / pap
        waxpby(1.0, x, alpha, p, x)
        waxpby(1.0, r, -alpha, ap, r)
        hist.append(math.sqrt(dot(r, r)) / scale)
        if hist[-1] <= tol:
            done = True
            break
        mg_vcycle(levels, 0, r, z)
        rtz_new = dot(r, z)
        waxpby(1.0, z, rtz_new / rtz, p, p)
        rtz = rtz_new
    return OCgResult(x, it, np.asarray(hist), done)
