"""Format-dispatched kernels on the B200 (kernels.py:1-337 of the reference).

Every compute call lands in libdynsparse_b200.so:

  spmv / spmv_add  -> ds_spmv (one ds_matrix descriptor, C-side format switch)
  dot              -> ds_dot (deterministic fixed-order tree)
  waxpby           -> ds_waxpby (two rounded products, one rounded add)
  reduce / scan    -> ds_scan (exact sequential np.cumsum order)
  extract/update_diagonal -> ds_extract_diag_* / ds_update_diag_* / ds_dia_diag_column

Bit-exactness vs the reference: CSR, DIA and sorted-COO SpMV, spmv_add,
waxpby, scan/reduce and the diagonal ops are bitwise identical; unsorted COO
SpMV uses atomics (within 1e-13, like the reference's threaded COO); dot is
a fixed tree (the reference's np.dot bits depend on the BLAS thread count).

Memory spaces: DEVICE operands run in place on their device (current torch
stream).  HOST operands (the reference's numpy containers) are staged to the
device, computed there and copied back, so the CUDA path is the only path.
``ExecBackend`` keeps the reference's contract (kinds "serial"/"threaded",
kernels.py:38-57); on the device the grid replaces the host thread pool.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import DimensionMismatch, StructurallyAbsentDiagonal
from .formats import (
    CooMatrix,
    CsrMatrix,
    DenseVector,
    DiaMatrix,
    DynamicMatrix,
    FormatId,
    MemorySpace,
)


@dataclass(frozen=True)
class ExecBackend:
    """Reference execution-backend record (kernels.py:38-57)."""

    kind: str = "serial"
    nthreads: int = 1

    def __post_init__(self):
        if self.kind not in ("serial", "threaded"):
            raise ValueError(f"unknown backend kind {self.kind!r}")
        if self.nthreads < 1:
            raise ValueError(f"nthreads must be >= 1, got {self.nthreads}")

    @staticmethod
    def serial() -> "ExecBackend":
        return ExecBackend("serial", 1)

    @staticmethod
    def threaded(nthreads: int) -> "ExecBackend":
        return ExecBackend("threaded", nthreads)


SERIAL = ExecBackend.serial()


def _resolve(a):
    return a.payload if isinstance(a, DynamicMatrix) else a


# ---------------------------------------------------------------------------
# device helpers
# ---------------------------------------------------------------------------

def _dev():
    from . import _device
    return _device


def _exec_device(*objs):
    """Device of the first DEVICE operand, else the current CUDA device."""
    for o in objs:
        if o is not None and getattr(o, "space", MemorySpace.HOST) == MemorySpace.DEVICE:
            return o.device
    return _dev().require_cuda()


def _on(obj, device):
    """obj itself if it already lives on ``device``, else a device copy."""
    from .datamove import to_device
    return to_device(obj, device)


def _key(*tensors):
    return tuple((t.data_ptr(), t._version, t.numel()) for t in tensors)


def csr_plan(m: CsrMatrix):
    """(long_rows tensor | None, n_long) for rows > 129 entries, cached per
    buffer version (ds_csr_analyze)."""
    k = ("plan",) + _key(m.row_offsets)
    hit = m._cache.get("plan")
    if hit is not None and hit[0] == k:
        return hit[1], hit[2]
    import torch
    D = _dev()
    lr, nl, ml = None, 0, 0
    if m.nrows > 0:
        buf = torch.empty(m.nrows, dtype=torch.int32, device=m.device)
        n_long, max_len = ctypes.c_int64(), ctypes.c_int32()
        with torch.cuda.device(m.device):
            _native.call("ds_csr_analyze", m.nrows, D.ptr(m.row_offsets), D.ptr(buf),
                         ctypes.byref(n_long), ctypes.byref(max_len), D.stream(m.device))
        nl, ml = int(n_long.value), int(max_len.value)
        # keep a valid pointer even when empty: non-NULL tells the C side the
        # matrix was analysed (rows > 129 are then handled by their own kernel)
        lr = buf[:max(nl, 1)].clone()
        # irregular rows (longer than the 33-entry paired fast path): bin rows
        # by length once, each bin then runs with its exact load rounds
        if int(max_len.value) > 33:
            perm = torch.empty(m.nrows, dtype=torch.int32, device=m.device)
            bins = (ctypes.c_int64 * 9)()
            with torch.cuda.device(m.device):
                _native.call("ds_csr_bins", m.nrows, D.ptr(m.row_offsets), D.ptr(perm), bins,
                             D.stream(m.device))
            # tile plan: row tiles + pairwise-leaf tiles of the long rows, with
            # the per-SpMV leaf-sum scratch at its end (ds_csr_tiles)
            cap = int(_native.load().ds_csr_tiles_capacity(m.nrows, m.nnz))
            tiles = torch.empty(cap, dtype=torch.int32, device=m.device)
            nt, used = ctypes.c_int64(), ctypes.c_int64()
            with torch.cuda.device(m.device):
                _native.call("ds_csr_tiles", m.nrows, D.ptr(m.row_offsets), D.ptr(tiles), cap,
                             ctypes.byref(nt), ctypes.byref(used), D.stream(m.device))
            m._cache["bins"] = (k, perm, list(bins), tiles[:int(used.value)].clone(),
                                int(nt.value))
    m._cache["plan"] = (k, lr, nl)
    m._cache["max_len"] = (k, ml)
    return lr, nl


def csr_bins(m: CsrMatrix):
    """(perm tensor, bins[9]) when the matrix was binned, else None."""
    csr_plan(m)
    hit = m._cache.get("bins")
    k = ("plan",) + _key(m.row_offsets)
    if hit is not None and hit[0] == k:
        return hit[1:]
    return None


def coo_flags(m: CooMatrix) -> int:
    """bit0: rows nondecreasing; bit1: strictly (row, col) increasing."""
    k = ("flags",) + _key(m.row_indices, m.col_indices)
    hit = m._cache.get("flags")
    if hit is not None and hit[0] == k:
        return hit[1]
    import torch
    D = _dev()
    flags = ctypes.c_int32(3)
    if m.nnz > 1:
        with torch.cuda.device(m.device):
            _native.call("ds_coo_order_flags", m.nnz, D.ptr(m.row_indices),
                         D.ptr(m.col_indices), ctypes.byref(flags), D.stream(m.device))
    run = 0
    if (int(flags.value) & 1) and m.nnz > 0:
        # longest row of a row-sorted COO: picks the SpMV kernel (<= 27:
        # thread-per-row pipeline, else warp segments)
        mr = ctypes.c_int32(0)
        with torch.cuda.device(m.device):
            _native.call("ds_coo_max_run", m.nnz, D.ptr(m.row_indices), ctypes.byref(mr),
                         D.stream(m.device))
        run = int(mr.value)
    m._cache["flags"] = (k, int(flags.value))
    m._cache["max_run"] = (k, run)
    return int(flags.value)


def coo_max_run(m: CooMatrix) -> int:
    """Longest run of equal row indices (0 unless rows are sorted)."""
    coo_flags(m)
    return m._cache["max_run"][1]


def coo_long_runs(m: CooMatrix):
    """(int32 tensor of (start, end) pairs, count) of the rows longer than the
    long-run kernel's threshold, for a row-sorted COO; (None, 0) otherwise.
    Cached per buffer version (ds_coo_long_runs)."""
    k = ("runs",) + _key(m.row_indices, m.col_indices)
    hit = m._cache.get("runs")
    if hit is not None and hit[0] == k:
        return hit[1], hit[2]
    import torch
    D = _dev()
    runs, cnt = None, 0
    thr = int(_native.load().ds_coo_long_run_threshold())
    if (coo_flags(m) & 1) and coo_max_run(m) > thr and \
            not os.environ.get("DS_COO_NO_LONG_RUNS"):
        cap = m.nnz // thr + 1
        buf = torch.empty(2 * cap, dtype=torch.int32, device=m.device)
        n = ctypes.c_int64(0)
        with torch.cuda.device(m.device):
            _native.call("ds_coo_long_runs", m.nnz, D.ptr(m.row_indices), thr, D.ptr(buf), cap,
                         ctypes.byref(n), D.stream(m.device))
        cnt = int(n.value)
        runs = buf[:2 * max(cnt, 1)].clone() if cnt else None
    m._cache["runs"] = (k, runs, cnt)
    return runs, cnt


def descriptor(m) -> _native.DsMatrix:
    """ds_matrix for a DEVICE container (the C-side dispatch record)."""
    m = _resolve(m)
    D = _dev()
    d = _native.DsMatrix()
    d.nrows, d.ncols = m.nrows, m.ncols
    D.check_dims(m.nrows, m.ncols)
    if isinstance(m, CsrMatrix):
        d.format, d.nnz = int(FormatId.CSR), m.nnz
        d.idx0, d.idx1, d.values = D.ptr(m.row_offsets), D.ptr(m.col_indices), D.ptr(m.values)
        lr, nl = csr_plan(m)
        d.long_rows, d.n_long = (lr.data_ptr() if lr is not None else None), nl
        d.max_row_len = m._cache["max_len"][1]
        b = csr_bins(m)
        if b is not None:
            d.row_perm = b[0].data_ptr()
            for i in range(len(d.bins)):
                d.bins[i] = b[1][i]
            if os.environ.get("DS_CSR_TILES", "1") != "0":
                d.tiles, d.ntiles = b[2].data_ptr(), b[3]
    elif isinstance(m, CooMatrix):
        d.format, d.nnz = int(FormatId.COO), m.nnz
        d.idx0, d.idx1, d.values = D.ptr(m.row_indices), D.ptr(m.col_indices), D.ptr(m.values)
        d.rows_sorted = coo_flags(m) & 1
        d.max_row_len = coo_max_run(m)
        runs, cnt = coo_long_runs(m)
        if runs is not None:
            d.long_rows, d.n_long = runs.data_ptr(), cnt
    elif isinstance(m, DiaMatrix):
        d.format, d.ndiags = int(FormatId.DIA), m.ndiags
        d.idx0, d.values = D.ptr(m.offsets), D.ptr(m.values)
    else:
        raise TypeError(f"not a sparse container: {type(m).__name__}")
    return d


def _dia_count_nonzero(m: DiaMatrix) -> int:
    import torch
    D = _dev()
    out = ctypes.c_int64()
    with torch.cuda.device(m.device):
        _native.call("ds_dia_count_nonzero", m.nrows, m.ncols, m.ndiags, D.ptr(m.offsets),
                     D.ptr(m.values), ctypes.byref(out), D.stream(m.device))
    return int(out.value)


def _device_vec(v: DenseVector, device):
    """(device tensor, writeback) for a possibly-HOST vector."""
    if v.space == MemorySpace.DEVICE and v.device == device:
        return v.data, None
    import torch
    if v.space == MemorySpace.DEVICE:
        t = v.data.to(device)
    else:
        t = torch.from_numpy(np.ascontiguousarray(v.data)).to(device)

    def writeback(t=t, v=v):
        if v.space == MemorySpace.HOST:
            v.data[:] = t.cpu().numpy()
        else:
            v.data.copy_(t)
    return t, writeback


# ---------------------------------------------------------------------------
# SpMV (kernels.py:166-198)
# ---------------------------------------------------------------------------

def _spmv(a, x: DenseVector, y: DenseVector, accumulate: int) -> None:
    import torch
    mat = _resolve(a)
    if x.length != mat.ncols:
        raise DimensionMismatch(f"x length {x.length} != ncols {mat.ncols}")
    if y.length != mat.nrows:
        raise DimensionMismatch(f"y length {y.length} != nrows {mat.nrows}")
    dev = _exec_device(mat, x, y)
    A = _on(mat, dev)
    xt, _ = _device_vec(x, dev)
    yt, wb = _device_vec(y, dev)
    D = _dev()
    d = descriptor(A)
    with torch.cuda.device(dev):
        _native.call("ds_spmv", ctypes.byref(d), D.ptr(xt), D.ptr(yt), accumulate,
                     D.stream(dev))
    if wb is not None:
        wb()


def prepared_spmv(a, x: DenseVector, y: DenseVector, accumulate: int):
    """Resolve, validate and build the descriptor once; return a launcher that
    only enqueues the kernel(s) (two ctypes calls' worth of host time), for
    timing loops whose CUDA events must bracket device work, not Python.
    DEVICE containers only."""
    import torch
    mat = _resolve(a)
    if x.length != mat.ncols:
        raise DimensionMismatch(f"x length {x.length} != ncols {mat.ncols}")
    if y.length != mat.nrows:
        raise DimensionMismatch(f"y length {y.length} != nrows {mat.nrows}")
    dev = _exec_device(mat, x, y)
    if not (isinstance(x.data, torch.Tensor) and isinstance(y.data, torch.Tensor)):
        raise TypeError("prepared_spmv needs DEVICE vectors")
    D = _dev()
    d = descriptor(_on(mat, dev))
    xp, yp, st = D.ptr(x.data), D.ptr(y.data), D.stream(dev)
    lib = _native.load()

    def launch():
        _native.check(lib.ds_spmv(ctypes.byref(d), xp, yp, accumulate, st))
    launch.keep = (d, x, y, mat)   # descriptor and buffers outlive the launcher
    return launch


def spmv(backend: ExecBackend, a, x: DenseVector, y: DenseVector) -> None:
    """y = A x, overwriting y (kernels.py:173-186)."""
    _spmv(a, x, y, 0)


def spmv_add(backend: ExecBackend, a, x: DenseVector, y: DenseVector) -> None:
    """y += A x (the remote-part accumulate, kernels.py:189-198)."""
    _spmv(a, x, y, 1)


multiply = spmv  # Morpheus's name for the operation


# ---------------------------------------------------------------------------
# dense-vector kernels (kernels.py:205-235)
# ---------------------------------------------------------------------------

def dot(backend: ExecBackend, x: DenseVector, y: DenseVector) -> float:
    """x . y; 0.0 for empty vectors (kernels.py:205-209)."""
    import torch
    if x.length != y.length:
        raise DimensionMismatch(f"lengths differ: {x.length} vs {y.length}")
    dev = _exec_device(x, y)
    xt, _ = _device_vec(x, dev)
    yt, _ = _device_vec(y, dev)
    D = _dev()
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        _native.call("ds_dot", x.length, D.ptr(xt), D.ptr(yt), D.ptr(out),
                     D.ptr(D.workspace(dev)), D.stream(dev))
    return float(out.item())


def waxpby(backend: ExecBackend, alpha: float, x: DenseVector, beta: float, y: DenseVector,
           w: DenseVector) -> None:
    """w = alpha*x + beta*y; w may alias x or y (kernels.py:212-219)."""
    import torch
    if not x.length == y.length == w.length:
        raise DimensionMismatch(f"lengths differ: x={x.length} y={y.length} w={w.length}")
    dev = _exec_device(w, x, y)
    xt, _ = _device_vec(x, dev)
    yt, _ = _device_vec(y, dev)
    if w is x:
        wt, wb = xt, None
    elif w is y:
        wt, wb = yt, None
    else:
        wt, wb = _device_vec(w, dev)
    D = _dev()
    with torch.cuda.device(dev):
        _native.call("ds_waxpby", w.length, float(alpha), D.ptr(xt), float(beta), D.ptr(yt),
                     D.ptr(wt), D.stream(dev))
    if w.space == MemorySpace.HOST and (w is x or w is y):
        w.data[:] = wt.cpu().numpy()
    elif wb is not None:
        wb()


def reduce(backend: ExecBackend, x: DenseVector) -> float:
    """Sum in sequential prefix order, == scan(x)[-1] exactly (kernels.py:222-230)."""
    import torch
    if x.length == 0:
        return 0.0
    dev = _exec_device(x)
    xt, _ = _device_vec(x, dev)
    D = _dev()
    total = torch.zeros(1, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        _native.call("ds_scan", x.length, D.ptr(xt), None, D.ptr(total), D.stream(dev))
    return float(total.item())


def scan(backend: ExecBackend, x: DenseVector) -> DenseVector:
    """Inclusive prefix sums (np.cumsum order) in x's memory space."""
    import torch
    dev = _exec_device(x)
    xt, _ = _device_vec(x, dev)
    D = _dev()
    out = torch.empty(x.length, dtype=torch.float64, device=dev)
    if x.length:
        with torch.cuda.device(dev):
            _native.call("ds_scan", x.length, D.ptr(xt), D.ptr(out), None, D.stream(dev))
    if x.space == MemorySpace.HOST:
        return DenseVector(out.cpu().numpy())
    return DenseVector(out)


# ---------------------------------------------------------------------------
# diagonal extract / update (kernels.py:242-337)
# ---------------------------------------------------------------------------

def _dia_main(m: DiaMatrix):
    offs = m.offsets if m.space == MemorySpace.HOST else m.offsets.cpu().numpy()
    hit = np.flatnonzero(np.asarray(offs) == 0)
    return int(hit[0]) if hit.size else None


def extract_diagonal(a) -> DenseVector:
    """Main diagonal, length min(nrows, ncols); absent entries read 0.0."""
    import torch
    mat = _resolve(a)
    n = min(mat.nrows, mat.ncols)
    dev = _exec_device(mat)
    A = _on(mat, dev)
    D = _dev()
    out = torch.zeros(n, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        st = D.stream(dev)
        if n == 0:
            pass
        elif isinstance(A, CsrMatrix):
            _native.call("ds_extract_diag_csr", A.nrows, A.ncols, D.ptr(A.row_offsets),
                         D.ptr(A.col_indices), D.ptr(A.values), D.ptr(out), st)
        elif isinstance(A, CooMatrix):
            _native.call("ds_extract_diag_coo", A.nrows, A.ncols, A.nnz, D.ptr(A.row_indices),
                         D.ptr(A.col_indices), D.ptr(A.values), D.ptr(out), st)
        else:
            j0 = _dia_main(A)
            if j0 is not None:
                _native.call("ds_dia_diag_column", n, A.ndiags, j0, D.ptr(A.values), D.ptr(out),
                             0, st)
    if mat.space == MemorySpace.HOST:
        return DenseVector(out.cpu().numpy())
    return DenseVector(out)


def update_diagonal(a, d: DenseVector) -> None:
    """Overwrite A(i,i) = d[i] keeping the sparsity; StructurallyAbsentDiagonal
    names the first missing row (kernels.py:325-337)."""
    import torch
    from .datamove import deep_copy
    mat = _resolve(a)
    n = min(mat.nrows, mat.ncols)
    if d.length != n:
        raise DimensionMismatch(f"diagonal length {d.length} != min(dims) = {n}")
    if n == 0:
        return
    dev = _exec_device(mat, d)
    A = _on(mat, dev)
    dt, _ = _device_vec(d, dev)
    D = _dev()
    missing = ctypes.c_int64(-1)
    with torch.cuda.device(dev):
        st = D.stream(dev)
        if isinstance(A, CsrMatrix):
            rc = _native.load().ds_update_diag_csr(A.nrows, A.ncols, D.ptr(A.row_offsets),
                                                   D.ptr(A.col_indices), D.ptr(A.values),
                                                   D.ptr(dt), ctypes.byref(missing), st)
        elif isinstance(A, CooMatrix):
            rc = _native.load().ds_update_diag_coo(A.nrows, A.ncols, A.nnz,
                                                   D.ptr(A.row_indices), D.ptr(A.col_indices),
                                                   D.ptr(A.values), D.ptr(dt),
                                                   ctypes.byref(missing), st)
        else:
            j0 = _dia_main(A)
            if j0 is None:
                raise StructurallyAbsentDiagonal(0)
            rc = _native.load().ds_dia_diag_column(n, A.ndiags, j0, D.ptr(A.values), D.ptr(dt),
                                                   1, st)
    if rc == _native.DS_ERR_STRUCTURALLY_ABSENT_DIAG:
        raise StructurallyAbsentDiagonal(int(missing.value))
    _native.check(rc)
    if A is not mat:  # HOST container: copy the updated values back
        deep_copy(A, mat)
