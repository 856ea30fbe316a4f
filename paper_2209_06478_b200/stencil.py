"""27-point stencil problem, 3-D block decomposition and halo exchange
(stencil.py:1-319 of the reference).

* ``generate_problem`` builds every partition's system exactly as the
  reference (diagonal 26, off-diagonals -1, x-fastest local numbering,
  rank = cx + px*(cy + py*cz), ghosts numbered by (owner, owner-local),
  columns sorted per row, b = row sums).  Integer-exact: HOST space runs
  numpy, ``space=MemorySpace.DEVICE`` runs the generator kernels on the GPU
  (ds_stencil_*) -- bitwise the same arrays.
* ``exchange_halo`` is a set of device gathers: each neighbour's send list
  is gathered straight into the receiver's contiguous ghost slice
  (ds_gather); across processes the same plan drives NCCL (dist.py).
* ``distributed_spmv`` = exchange, then local SpMV + remote spmv_add per
  partition on the device; optional per-partition timing uses CUDA events.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import DimensionMismatch
from .formats import CsrMatrix, DenseVector, DynamicMatrix, MemorySpace
from .kernels import ExecBackend, spmv, spmv_add

STENCIL_DIAG = 26.0
STENCIL_OFF_DIAG = -1.0


@dataclass(frozen=True)
class GridSpec:
    """Per-partition extents nx, ny, nz and the partition grid px, py, pz
    (stencil.py:33-68)."""

    nx: int
    ny: int
    nz: int
    px: int = 1
    py: int = 1
    pz: int = 1

    def __post_init__(self):
        for name in ("nx", "ny", "nz", "px", "py", "pz"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1, got {getattr(self, name)}")

    @property
    def local_points(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def npartitions(self) -> int:
        return self.px * self.py * self.pz

    @property
    def global_dims(self) -> tuple[int, int, int]:
        return (self.nx * self.px, self.ny * self.py, self.nz * self.pz)

    @property
    def global_points(self) -> int:
        gx, gy, gz = self.global_dims
        return gx * gy * gz


@dataclass
class HaloExchange:
    """One neighbour's share of a partition's ghosts (stencil.py:71-82)."""

    neighbor: int
    send_local_indices: np.ndarray
    recv_ghost_slots: np.ndarray


@dataclass
class HaloPlan:
    """Ghost slots local_n .. local_n + ghost_count - 1 (stencil.py:85-93)."""

    ghost_count: int
    exchanges: list[HaloExchange] = field(default_factory=list)


@dataclass
class PartitionData:
    """One partition's system, plan and index maps (stencil.py:96-107)."""

    rank: int
    coords: tuple[int, int, int]
    a_full: CsrMatrix
    b: DenseVector
    xexact: DenseVector
    halo: HaloPlan
    local_to_global: np.ndarray
    ghost_to_global: np.ndarray
    device_cache: dict = field(default_factory=dict, repr=False, compare=False)


@dataclass
class PartitionedProblem:
    spec: GridSpec
    partitions: list[PartitionData]

    @property
    def npartitions(self) -> int:
        return len(self.partitions)


@dataclass
class SplitMatrix:
    """local: square over owned columns; remote: rows x ghosts, columns
    re-based to 0 (stencil.py:122-132)."""

    local: DynamicMatrix
    remote: DynamicMatrix


_STEPS = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]


def _partition(spec: GridSpec, rank: int) -> PartitionData:
    """Assemble one partition (the reference's per-rank body, stencil.py:168-251).

    Columns of each row are laid out in a (n, 27) table -- owned neighbours
    by owner-local index, ghosts by n + their rank in the sorted
    (owner, owner-local) key list -- and sorted along the row, which gives
    exactly the reference's lexsort((cols, rows)) order."""
    nx, ny, nz, px, py, pz = spec.nx, spec.ny, spec.nz, spec.px, spec.py, spec.pz
    gnx, gny, gnz = spec.global_dims
    n = spec.local_points
    cx, cy, cz = rank % px, (rank // px) % py, rank // (px * py)
    ids = np.arange(n, dtype=np.int64)
    gx = ids % nx + cx * nx
    gy = (ids // nx) % ny + cy * ny
    gz = ids // (nx * ny) + cz * nz
    sentinel = np.iinfo(np.int64).max
    key = np.full((n, 27), sentinel, dtype=np.int64)   # owner*n + owner_local
    for t, (dx, dy, dz) in enumerate(_STEPS):
        tx, ty, tz = gx + dx, gy + dy, gz + dz
        ok = (tx >= 0) & (tx < gnx) & (ty >= 0) & (ty < gny) & (tz >= 0) & (tz < gnz)
        ox, oy, oz = tx // nx, ty // ny, tz // nz
        owner = ox + px * (oy + py * oz)
        oloc = (tx - ox * nx) + nx * ((ty - oy * ny) + ny * (tz - oz * nz))
        key[:, t] = np.where(ok, owner * n + oloc, sentinel)
    valid = key != sentinel
    own = valid & (key // n == rank)
    ghost = valid & ~own
    ghost_keys = np.unique(key[ghost])
    col = np.full((n, 27), sentinel, dtype=np.int64)
    col[own] = key[own] - rank * n
    if ghost_keys.size:
        col[ghost] = n + np.searchsorted(ghost_keys, key[ghost])
    col.sort(axis=1)
    counts = valid.sum(axis=1)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    cols = col[col != sentinel]
    rows = np.repeat(ids, counts)
    vals = np.where(cols == rows, STENCIL_DIAG, STENCIL_OFF_DIAG)
    b = (27.0 - counts).astype(np.float64)   # 26 - (count - 1): exact row sums
    g_owner, g_local = ghost_keys // n, ghost_keys % n
    exchanges = []
    for q in np.unique(g_owner).tolist():
        sel = np.flatnonzero(g_owner == q)
        exchanges.append(HaloExchange(int(q), g_local[sel].copy(), n + sel))
    qx, qy, qz = g_owner % px, (g_owner // px) % py, g_owner // (px * py)
    g2g = ((g_local % nx + qx * nx)
           + gnx * (((g_local // nx) % ny + qy * ny) + gny * (g_local // (nx * ny) + qz * nz)))
    return PartitionData(
        rank=rank, coords=(cx, cy, cz),
        a_full=CsrMatrix(n, n + int(ghost_keys.size), offsets, cols, vals),
        b=DenseVector(b), xexact=DenseVector.ones(n),
        halo=HaloPlan(int(ghost_keys.size), exchanges),
        local_to_global=gx + gnx * (gy + gny * gz), ghost_to_global=g2g)


def halo_send_lists(spec: GridSpec, rank: int) -> dict[int, np.ndarray]:
    """What this rank must SEND each neighbour: q's ghosts owned by ``rank``.

    The stencil is symmetric, so my point i is a ghost of q iff one of i's
    27 neighbours is owned by q; q numbers its ghosts by (owner, owner-local)
    ascending (stencil.py:198-209), so the list is my local indices in
    ascending order -- exactly q's HaloExchange.send_local_indices for me
    (stencil.py:221-230), computed without generating q's partition."""
    nx, ny, nz, px, py, pz = spec.nx, spec.ny, spec.nz, spec.px, spec.py, spec.pz
    gnx, gny, gnz = spec.global_dims
    n = spec.local_points
    cx, cy, cz = rank % px, (rank // px) % py, rank // (px * py)
    ids = np.arange(n, dtype=np.int64)
    gx = ids % nx + cx * nx
    gy = (ids // nx) % ny + cy * ny
    gz = ids // (nx * ny) + cz * nz
    per_owner: dict[int, list[np.ndarray]] = {}
    for dx, dy, dz in _STEPS:
        tx, ty, tz = gx + dx, gy + dy, gz + dz
        ok = (tx >= 0) & (tx < gnx) & (ty >= 0) & (ty < gny) & (tz >= 0) & (tz < gnz)
        owner = (tx // nx) + px * ((ty // ny) + py * (tz // nz))
        far = ok & (owner != rank)
        if not far.any():
            continue
        for q in np.unique(owner[far]).tolist():
            per_owner.setdefault(int(q), []).append(ids[far & (owner == q)])
    return {q: np.unique(np.concatenate(v)) for q, v in sorted(per_owner.items())}


def _partition_device(spec: GridSpec, rank: int, device) -> PartitionData:
    """Device-side generation (ds_stencil_begin / ds_stencil_finish): the
    matrix, b and the sorted ghost keys are produced by kernels; the halo
    plan and the two index maps follow on the host from the ghost keys
    (O(ghosts) + O(n) integer arithmetic)."""
    import ctypes

    import torch
    from . import _device
    dev = _device.require_cuda(device)
    n = spec.local_points
    lib = _native.load()
    job = ctypes.c_void_p()
    nnz, ng = ctypes.c_int64(), ctypes.c_int64()
    with torch.cuda.device(dev):
        st = _device.stream(dev)
        _native.check(lib.ds_stencil_begin(spec.nx, spec.ny, spec.nz, spec.px, spec.py, spec.pz,
                                           rank, st, ctypes.byref(job), ctypes.byref(nnz),
                                           ctypes.byref(ng)))
        i32 = dict(dtype=torch.int32, device=dev)
        f64 = dict(dtype=torch.float64, device=dev)
        off = torch.empty(n + 1, **i32)
        cols = torch.empty(int(nnz.value), **i32)
        vals = torch.empty(int(nnz.value), **f64)
        b = torch.empty(n, **f64)
        keys = torch.empty(max(int(ng.value), 1), dtype=torch.int64, device=dev)
        _native.check(lib.ds_stencil_finish(job, off.data_ptr(), cols.data_ptr(),
                                            vals.data_ptr(), b.data_ptr(), keys.data_ptr()))
        ghost_keys = keys[:int(ng.value)].cpu().numpy()
    nx, ny, nz, px, py, pz = spec.nx, spec.ny, spec.nz, spec.px, spec.py, spec.pz
    gnx, gny, gnz = spec.global_dims
    cx, cy, cz = rank % px, (rank // px) % py, rank // (px * py)
    g_owner, g_local = ghost_keys // n, ghost_keys % n
    exchanges = []
    for q in np.unique(g_owner).tolist():
        sel = np.flatnonzero(g_owner == q)
        exchanges.append(HaloExchange(int(q), g_local[sel].copy(), n + sel))
    ids = np.arange(n, dtype=np.int64)
    gx = ids % nx + cx * nx
    gy = (ids // nx) % ny + cy * ny
    gz = ids // (nx * ny) + cz * nz
    qx, qy, qz = g_owner % px, (g_owner // px) % py, g_owner // (px * py)
    g2g = ((g_local % nx + qx * nx)
           + gnx * (((g_local // nx) % ny + qy * ny) + gny * (g_local // (nx * ny) + qz * nz)))
    return PartitionData(
        rank=rank, coords=(cx, cy, cz),
        a_full=CsrMatrix(n, n + int(ghost_keys.size), off, cols, vals, MemorySpace.DEVICE),
        b=DenseVector(b), xexact=DenseVector.ones(n, MemorySpace.DEVICE, dev),
        halo=HaloPlan(int(ghost_keys.size), exchanges),
        local_to_global=gx + gnx * (gy + gny * gz), ghost_to_global=g2g)


def _to_space(part: PartitionData, space, device) -> PartitionData:
    if space is None or MemorySpace(space) == MemorySpace.HOST:
        return part
    from .datamove import to_device
    part.a_full = to_device(part.a_full, device)
    part.b = to_device(part.b, device)
    part.xexact = to_device(part.xexact, device)
    return part


def generate_problem(spec: GridSpec, space: MemorySpace | None = None, device=None,
                     ranks=None) -> PartitionedProblem:
    """Every partition's stencil system (stencil.py:143-253).  ``ranks``
    restricts generation to a subset (one rank per process); ``space``
    places matrices/vectors on the device."""
    which = range(spec.npartitions) if ranks is None else list(ranks)
    parts = [generate_partition(spec, r, space, device) for r in which]
    return PartitionedProblem(spec=spec, partitions=parts)


def generate_partition(spec: GridSpec, rank: int, space: MemorySpace | None = None,
                       device=None) -> PartitionData:
    """One partition.  DEVICE space: generated by kernels on the device
    (set DS_HOST_GENERATOR=1 to build on the host and upload instead)."""
    import os
    if space is not None and MemorySpace(space) == MemorySpace.DEVICE and \
            not os.environ.get("DS_HOST_GENERATOR"):
        return _partition_device(spec, rank, device)
    return _to_space(_partition(spec, rank), space, device)


def _split_host(a: CsrMatrix, ghost_count: int):
    n = a.nrows
    inner = a.col_indices < n
    row_of = np.repeat(np.arange(n, dtype=np.int64), np.diff(a.row_offsets))

    def part(mask, ncols, shift):
        off = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(row_of[mask], minlength=n), out=off[1:])
        return CsrMatrix(n, ncols, off, a.col_indices[mask] - shift, a.values[mask])

    return part(inner, n, 0), part(~inner, ghost_count, n)


def split_local_remote(problem: PartitionedProblem, partition: int) -> SplitMatrix:
    """Cut a_full into local (cols < n) and remote (cols >= n, shifted) CSR
    parts, both CSR-active DynamicMatrix (stencil.py:256-277).  Integer
    setup; DEVICE matrices are split and returned on their device."""
    part = problem.partitions[partition]
    a = part.a_full
    if a.space == MemorySpace.HOST:
        loc, rem = _split_host(a, part.halo.ghost_count)
    else:
        loc, rem = _split_device(a, part.halo.ghost_count)
    return SplitMatrix(local=DynamicMatrix(loc), remote=DynamicMatrix(rem))


def _split_device(a: CsrMatrix, ghost_count: int):
    """ds_csr_split_count / ds_csr_split_fill on a DEVICE CSR."""
    import ctypes

    import torch
    from . import _device
    n, dev = a.nrows, a.device
    lib = _native.load()
    i32 = dict(dtype=torch.int32, device=dev)
    f64 = dict(dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        st = _device.stream(dev)
        loc_off = torch.empty(n + 1, **i32)
        nl = ctypes.c_int64()
        _native.check(lib.ds_csr_split_count(n, n, a.row_offsets.data_ptr(),
                                             _device.ptr(a.col_indices), loc_off.data_ptr(),
                                             ctypes.byref(nl), st))
        nl = int(nl.value)
        nr = a.nnz - nl
        lc, lv = torch.empty(nl, **i32), torch.empty(nl, **f64)
        ro, rc, rv = torch.empty(n + 1, **i32), torch.empty(nr, **i32), torch.empty(nr, **f64)
        _native.check(lib.ds_csr_split_fill(n, n, a.nnz, a.row_offsets.data_ptr(),
                                            _device.ptr(a.col_indices), _device.ptr(a.values),
                                            loc_off.data_ptr(), nl, _device.ptr(lc),
                                            _device.ptr(lv), ro.data_ptr(), _device.ptr(rc),
                                            _device.ptr(rv), st))
    return (CsrMatrix(n, n, loc_off, lc, lv, MemorySpace.DEVICE),
            CsrMatrix(n, ghost_count, ro, rc, rv, MemorySpace.DEVICE))


# ---------------------------------------------------------------------------
# device halo plan
# ---------------------------------------------------------------------------

def device_halo(part: PartitionData, device):
    """[(neighbor, count, send_idx int32 tensor, recv_start)] on ``device``;
    recv_start is the ABSOLUTE slot (>= n) of the neighbour's first ghost.
    Recv slots are one contiguous slice per neighbour (ghosts are numbered by
    owner), so the gather writes straight into x[n + start : ...]."""
    import torch
    key = ("halo", str(device))
    hit = part.device_cache.get(key)
    if hit is not None:
        return hit
    from . import _device
    out = []
    for ex in part.halo.exchanges:
        slots = np.asarray(ex.recv_ghost_slots, dtype=np.int64)
        cnt = int(slots.size)
        start = int(slots[0]) if cnt else 0
        if cnt and not np.array_equal(slots, np.arange(start, start + cnt)):
            raise NotImplementedError("non-contiguous ghost slots are not supported")
        idx = _device.to_index_tensor(np.asarray(ex.send_local_indices), device)
        out.append((int(ex.neighbor), cnt, idx, start))
    part.device_cache[key] = out
    torch.cuda.synchronize(device)
    return out


def _exchange_device(problem: PartitionedProblem, xs: list) -> None:
    import torch
    from . import _device
    for part, x in zip(problem.partitions, xs):
        dev = x.data.device
        with torch.cuda.device(dev):
            st = _device.stream(dev)
            for q, cnt, idx, start in device_halo(part, dev):
                if cnt == 0:
                    continue
                src = xs[q].data
                dst = x.data[start:start + cnt]
                _native.call("ds_gather", cnt, idx.data_ptr(), src.data_ptr(), dst.data_ptr(), st)


def _check_lengths(problem, xs):
    n = problem.spec.local_points
    for part, x in zip(problem.partitions, xs):
        want = n + part.halo.ghost_count
        if x.length != want:
            raise DimensionMismatch(f"partition {part.rank}: vector length {x.length} != {want}")


def _staged(vectors):
    """Device views of the vectors (HOST ones uploaded) + write-back hook."""
    from .datamove import to_device
    from .formats import MemorySpace as MS
    dev_vecs, backs = [], []
    for v in vectors:
        if v.space == MS.DEVICE:
            dev_vecs.append(v)
        else:
            d = to_device(v)
            dev_vecs.append(d)
            backs.append((v, d))

    def writeback():
        for h, d in backs:
            h.data[:] = d.data.cpu().numpy()
    return dev_vecs, writeback


def exchange_halo(problem: PartitionedProblem, xs: list[DenseVector]) -> None:
    """Fill each partition's ghost slots from the owners (stencil.py:280-295)."""
    _check_lengths(problem, xs)
    dxs, wb = _staged(xs)
    _exchange_device(problem, dxs)
    wb()


def distributed_spmv(backend: ExecBackend, problem: PartitionedProblem,
                     splits: list[SplitMatrix], xs: list[DenseVector], ys: list[DenseVector],
                     per_partition_ns: list[int] | None = None) -> None:
    """y_k = local_k x_owned + remote_k x_ghost after the halo exchange
    (stencil.py:298-319).  per_partition_ns receives each partition's
    device compute time (exchange excluded) from CUDA events."""
    import torch
    _check_lengths(problem, xs)
    dxs, wbx = _staged(xs)
    dys, wby = _staged(ys)
    _exchange_device(problem, dxs)
    n = problem.spec.local_points
    events = []
    for k, split in enumerate(splits):
        dev = dxs[k].data.device
        if per_partition_ns is not None:
            # prepare first, so the events bracket the kernels, not Python
            from .kernels import prepared_spmv
            lo = prepared_spmv(split.local, DenseVector(dxs[k].data[:n]), dys[k], 0)
            ro = prepared_spmv(split.remote, DenseVector(dxs[k].data[n:]), dys[k], 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream(dev))
            lo()
            ro()
            e1.record(torch.cuda.current_stream(dev))
            events.append((k, e0, e1))
            continue
        spmv(backend, split.local, DenseVector(dxs[k].data[:n]), dys[k])
        spmv_add(backend, split.remote, DenseVector(dxs[k].data[n:]), dys[k])
    if per_partition_ns is not None:
        for k, e0, e1 in events:
            e1.synchronize()
            per_partition_ns[k] = int(round(e0.elapsed_time(e1) * 1e6))
    wbx()
    wby()
