"""One partition per process: halo exchange and global dots over NCCL.

The reference simulates MPI ranks as list entries in one process
(stencil.py:9-15); on the B200 node each rank is a process driving one GPU
(torch.distributed only bootstraps: it broadcasts the NCCL unique id).
Per CG iteration (solver.py:170-188):

    halo      pack kernels + one NCCL group of send/recv pairs (side stream),
              overlapped with the local SpMV on the compute stream
    Ap        local SpMV; then remote spmv_add fused with the partial p.Ap
    p.Ap      ncclAllGather of the P partials, rank-ordered sum on device
    x, r      fused update + partial r.r; all-gather; finalize (history, beta)
    p         p = r + beta p

All of it is stream-ordered with device-side scalars, so one iteration is
captured once as a CUDA graph (NCCL supports stream capture) and replayed.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .formats import DenseVector, MemorySpace
from .kernels import descriptor
from .stencil import GridSpec, PartitionData, SplitMatrix, halo_send_lists

PAP, RR = _native.DS_CG_STAGE_PAP, _native.DS_CG_STAGE_RR


@dataclass
class HaloSchedule:
    """Everything one rank needs to run the exchange: per neighbour (ascending
    rank) the send list, the receive count and the ABSOLUTE first ghost slot."""

    rank: int
    n: int
    peers: list[int]
    send_idx: list[np.ndarray]
    recv_counts: list[int]
    recv_starts: list[int]

    @classmethod
    def build(cls, spec: GridSpec, part: PartitionData) -> "HaloSchedule":
        sends = halo_send_lists(spec, part.rank)
        recvs = {ex.neighbor: ex for ex in part.halo.exchanges}
        n = spec.local_points
        peers = sorted(set(sends) | set(recvs))
        recv_counts, recv_starts, send_idx = [], [], []
        for q in peers:
            slots = np.asarray(recvs[q].recv_ghost_slots) if q in recvs else np.zeros(0, np.int64)
            if slots.size and not np.array_equal(slots, np.arange(slots[0], slots[0] + slots.size)):
                raise NotImplementedError("ghost slots of one owner must be contiguous")
            recv_counts.append(int(slots.size))
            recv_starts.append(int(slots[0]) if slots.size else n)
            send_idx.append(sends.get(q, np.zeros(0, np.int64)))
        return cls(part.rank, n, peers, send_idx, recv_counts, recv_starts)


def init_comm(device) -> tuple[int, int, int]:
    """NCCL communicator over the default torch.distributed group (unique id
    broadcast from rank 0).  Returns (comm handle, rank, world)."""
    import torch
    import torch.distributed as dist
    lib = _native.load()
    rank, world = dist.get_rank(), dist.get_world_size()
    nb = lib.ds_nccl_unique_id_bytes()
    buf = ctypes.create_string_buffer(nb)
    if rank == 0:
        _native.check(lib.ds_nccl_unique_id(buf, nb))
    obj = [buf.raw if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = ctypes.c_void_p()
    with torch.cuda.device(device):
        _native.check(lib.ds_nccl_comm_init(obj[0], world, rank, ctypes.byref(comm)))
    return comm.value, rank, world


class RankCG:
    """Device CG for this rank's partition; same driver interface as
    solver.CgEngine (setup / step / capture_step / replay / scalars)."""

    def __init__(self, spec: GridSpec, part: PartitionData, split: SplitMatrix, device,
                 tol: float, max_iters: int, comm=None, world: int | None = None):
        import torch
        from . import _device
        from .datamove import to_device
        self.dev = device
        if comm is None:
            comm, _, world = init_comm(device)
        self.comm, self.P = comm, int(world)
        self.spec, self.part = spec, part
        self.n = n = spec.local_points
        self.tol, self.max_iters = float(tol), int(max_iters)
        self.local = to_device(split.local.payload, device)
        self.remote = to_device(split.remote.payload, device)
        self.d_local = descriptor(self.local)
        # an empty remote part (world size 1) only adds +0.0: fold it into the
        # local kernel's epilogue (mode 2) instead of a pass over every row
        self.fold = self.remote.nnz == 0
        self.d_remote = None if self.fold else descriptor(self.remote)
        f64 = dict(dtype=torch.float64, device=device)
        g = part.halo.ghost_count
        # one allocation for the iteration's vectors (256-B aligned segments)
        # so one persisting-L2 window covers them (capture_step)
        seg = lambda m: (m + 31) // 32 * 32   # noqa: E731
        sizes = [seg(n + g), seg(n), seg(n), seg(n)]
        self.vec_block = torch.zeros(sum(sizes), **f64)
        o = [0, sizes[0], sizes[0] + sizes[1], sizes[0] + sizes[1] + sizes[2]]
        self.p_full = self.vec_block[o[0]:o[0] + n + g]
        self.p = self.p_full[:n]
        self.x = self.vec_block[o[1]:o[1] + n]
        self.r = self.vec_block[o[2]:o[2] + n]
        self.ap = self.vec_block[o[3]:o[3] + n]
        self.b = to_device(part.b, device).data
        self.scal = torch.zeros(_native.CG_SCALARS_BYTES // 8, **f64)
        self.hist = torch.zeros(self.max_iters + 1, **f64)
        self.mine = torch.zeros(4, **f64)              # [pap, rr, bb0, rr0] partials
        self.all = torch.zeros(4 * self.P, **f64)      # gathered, one row per stage
        self.lib = _native.load()
        self.ws = _device.workspace(device)
        sched = HaloSchedule.build(spec, part)
        self.sched = sched
        self.nnbr = len(sched.peers)
        self._send_idx = [_device.to_index_tensor(s, device) for s in sched.send_idx]
        total = sum(int(s.size) for s in sched.send_idx)
        self._send_buf = torch.zeros(max(total, 1), **f64)
        bufs, off = [], 0
        for s in sched.send_idx:
            bufs.append(self._send_buf.data_ptr() + 8 * off)
            off += int(s.size)
        arr = lambda ty, vals: (ty * max(len(vals), 1))(*vals)  # noqa: E731
        self._c_peers = arr(ctypes.c_int32, sched.peers)
        self._c_scount = arr(ctypes.c_int64, [int(s.size) for s in sched.send_idx])
        self._c_sidx = arr(ctypes.c_void_p, [t.data_ptr() if t.numel() else None
                                             for t in self._send_idx])
        self._c_sbuf = arr(ctypes.c_void_p, bufs)
        self._c_rcount = arr(ctypes.c_int64, sched.recv_counts)
        self._c_rstart = arr(ctypes.c_int64, sched.recv_starts)
        self.side = torch.cuda.Stream(device)
        self.graph = None
        self._marks = None

    # -- primitives -----------------------------------------------------------
    def _ck(self, rc):
        _native.check(rc)

    def _exchange(self, stream, guard) -> None:
        self._ck(self.lib.ds_halo_exchange(self.nnbr, self._c_peers, self._c_scount, self._c_sidx,
                                           self._c_sbuf, self._c_rcount, self._c_rstart,
                                           self.p_full.data_ptr(), guard, self.comm, stream))

    def _gather(self, k: int, stream) -> None:
        m = self.mine.data_ptr() + 8 * k
        a = self.all.data_ptr() + 8 * k * self.P
        self._ck(self.lib.ds_allgather_f64(m, a, 1, self.comm, stream))

    def _allp(self, k):
        return self.all.data_ptr() + 8 * k * self.P

    def _mine(self, k):
        return self.mine.data_ptr() + 8 * k

    # -- CG -------------------------------------------------------------------
    def setup(self, stream) -> None:
        lib, ws = self.lib, self.ws.data_ptr()
        self._exchange(stream, None)
        self._ck(lib.ds_cg_spmv_dot(ctypes.byref(self.d_local), self.p_full.data_ptr(),
                                    self.ap.data_ptr(), 2 if self.fold else 0, None, None, 0,
                                    None, None, None, 0, ws, stream))
        if not self.fold:
            self._ck(lib.ds_cg_spmv_dot(ctypes.byref(self.d_remote),
                                        self.p_full.data_ptr() + 8 * self.n, self.ap.data_ptr(),
                                        1, None, None, 0, None, None, None, 0, ws, stream))
        self._ck(lib.ds_cg_setup_residual(self.n, self.b.data_ptr(), self.ap.data_ptr(),
                                          self.r.data_ptr(), self.p.data_ptr(), self._mine(2),
                                          self._mine(3), ws, stream))
        self._gather(2, stream)
        self._gather(3, stream)
        self._ck(lib.ds_cg_setup_finalize(self.scal.data_ptr(), self._allp(2), self._allp(3),
                                          self.P, self.tol, self.max_iters,
                                          self.hist.data_ptr(), stream))

    def step(self, stream) -> None:
        """One iteration; the halo exchange runs on a side stream while the
        local SpMV (which reads owned entries only) runs on ``stream``."""
        import torch
        lib, ws = self.lib, self.ws.data_ptr()
        s, hist = self.scal.data_ptr(), self.hist.data_ptr()
        main = torch.cuda.ExternalStream(stream, device=self.dev)
        self.side.wait_stream(main)
        self._exchange(self.side.cuda_stream, s)
        if self._marks is not None:
            self._marks[1].record(main)
        if self.fold:   # world size 1: local SpMV + fused partition p.Ap
            self._ck(lib.ds_cg_spmv_dot(ctypes.byref(self.d_local), self.p_full.data_ptr(),
                                        self.ap.data_ptr(), 2, self.p.data_ptr(), self._mine(0),
                                        PAP, s, hist, None, 0, ws, stream))
            if self._marks is not None:
                self._marks[2].record(main)
            main.wait_stream(self.side)
        else:
            self._ck(lib.ds_cg_spmv_dot(ctypes.byref(self.d_local), self.p_full.data_ptr(),
                                        self.ap.data_ptr(), 0, None, None, 0, s, None, None, 0,
                                        ws, stream))
            if self._marks is not None:
                self._marks[2].record(main)
            main.wait_stream(self.side)
            self._ck(lib.ds_cg_spmv_dot(ctypes.byref(self.d_remote),
                                        self.p_full.data_ptr() + 8 * self.n, self.ap.data_ptr(), 1,
                                        self.p.data_ptr(), self._mine(0), PAP, s, hist, None, 0,
                                        ws, stream))
        self._gather(0, stream)
        # alpha from the rank-ordered sum of the gathered p.Ap, x/r update,
        # this partition's r.r -> all-gather -> history / beta / p update
        self._ck(lib.ds_cg_update_gathered(self.n, self.x.data_ptr(), self.r.data_ptr(),
                                           self.p.data_ptr(), self.ap.data_ptr(), s,
                                           self._allp(0), self.P, self._mine(1), ws, stream))
        self._gather(1, stream)
        self._ck(lib.ds_cg_direction_gathered(self.n, self.r.data_ptr(), self.p.data_ptr(), s,
                                              hist, self._allp(1), self.P, ws, stream))

    def scalars(self) -> _native.DsCgScalars:
        return _native.DsCgScalars.from_buffer_copy(self.scal.cpu().numpy().tobytes())

    def capture_step(self) -> None:
        """Capture one iteration (kernels + NCCL) as a CUDA graph; fall back
        to eager launches if this NCCL/driver combination refuses capture."""
        import torch
        from . import _device
        cap = torch.cuda.Stream(self.dev)
        with torch.cuda.stream(cap):
            ws = _device.workspace(self.dev)
        torch.cuda.synchronize(self.dev)
        saved, self.ws = self.ws, ws
        import os
        if os.environ.get("DS_CG_L2_PERSIST", "1") != "0":
            self._l2_persist = self.lib.ds_l2_persist(
                self.vec_block.data_ptr(), self.vec_block.numel() * 8, cap.cuda_stream) == 0
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g, stream=cap):
                self.step(cap.cuda_stream)
            self.graph = g
        except Exception:  # pragma: no cover - depends on the NCCL build
            self.graph = None
        finally:
            self.ws = saved

    def release_l2(self, stream) -> None:
        """Give the persisting-L2 carve-out back (set by capture_step)."""
        if getattr(self, "_l2_persist", False):
            self.lib.ds_l2_persist_reset(stream)
            self._l2_persist = False

    def replay(self) -> None:
        import torch
        if self.graph is not None:
            self.graph.replay()
        else:
            self.step(torch.cuda.current_stream(self.dev).cuda_stream)

    def launches_per_step(self) -> int:
        packs = sum(1 for s in self.sched.send_idx if s.size)
        return packs + (1 if self.fold else 2) + 2    # packs, SpMV(s), update, direction

    def time_spmv_in_steps(self, steps: int, stream_handle=None) -> dict:
        import torch
        st = torch.cuda.current_stream(self.dev)
        ev = []
        for _ in range(steps):
            a, b, c, d = (torch.cuda.Event(enable_timing=True) for _ in range(4))
            a.record(st)
            self._marks = (st, b, c)
            try:
                self.step(st.cuda_stream)
            finally:
                self._marks = None
            d.record(st)
            ev.append((a, b, c, d))
        torch.cuda.synchronize(self.dev)
        k = [b.elapsed_time(c) for _, b, c, _ in ev]
        s = [a.elapsed_time(d) for a, _, _, d in ev]
        return {"avg_ms": sum(k) / len(k), "step_ms": sum(s) / len(s), "launches": len(k)}

    @property
    def parts(self):
        return [self]

    def solve(self) -> tuple[DenseVector, int, np.ndarray, bool]:
        """Run to convergence (chunked graph replays) and return this rank's x."""
        import torch
        with torch.cuda.device(self.dev):
            st = torch.cuda.current_stream(self.dev).cuda_stream
            self.setup(st)
            sc = self.scalars()
            if not sc.done:
                self.capture_step()
                while True:
                    for _ in range(8):
                        self.replay()
                    sc = self.scalars()
                    if sc.done:
                        break
        it = int(sc.iter)
        if sc.done == 2:
            from .errors import BreakdownZeroCurvature
            raise BreakdownZeroCurvature(f"p'Ap = {sc.pap} at iteration {it + 1}")
        hist = self.hist[:it + 1].cpu().numpy().copy()
        return DenseVector(self.x), it, hist, sc.done == 1

    def solve_host(self, b_host: np.ndarray, iters: int, chunk: int = 8) -> np.ndarray:
        """End-to-end solve through host memory: b from a numpy array (pinned
        staging), setup, ``iters`` iterations (tolerance as configured), x back
        to a numpy array.  Reuses this engine's buffers and captured graph."""
        import torch
        with torch.cuda.device(self.dev):
            st = torch.cuda.current_stream(self.dev)
            pin = self.__dict__.get("_pin")
            if pin is None:
                pin = (torch.empty(self.n, dtype=torch.float64, pin_memory=True),
                       torch.empty(self.n, dtype=torch.float64, pin_memory=True))
                self._pin = pin
            pin[0].copy_(torch.from_numpy(np.ascontiguousarray(b_host)))   # multi-threaded
            self.b.copy_(pin[0], non_blocking=True)
            self.x.zero_()
            self.p.zero_()
            self.setup(st.cuda_stream)
            for _ in range(iters):
                self.replay()
            pin[1].copy_(self.x, non_blocking=True)
            st.synchronize()
            return torch.empty_like(pin[1]).copy_(pin[1]).numpy()

    def close(self) -> None:
        if self.comm:
            _native.check(self.lib.ds_nccl_comm_destroy(self.comm))
            self.comm = None


def rank_cg(spec: GridSpec, part: PartitionData, split: SplitMatrix, tol: float = 1e-9,
            max_iters: int = 500, device=None):
    """CG across processes, one partition per rank (torch.distributed must be
    initialised).  Returns (x_owned DenseVector, iterations, history, converged)."""
    from . import _device
    dev = _device.require_cuda(device)
    eng = RankCG(spec, part, split, dev, tol, max_iters)
    try:
        return eng.solve()
    finally:
        eng.close()


def profile_rank(part: PartitionData, split: SplitMatrix, reps: int = 20,
                 fill_limit: int | None = None) -> dict:
    """This rank's row of the tuner's TimingTable (tuner.py:53-120): every
    (local, remote) combination converted in place (wall time of a second,
    warm-pool conversion recorded -- the cost of runtime switching; the first
    also grows the memory pool), one warm-up, then the median
    of ``reps`` CUDA-event timings of local SpMV + remote spmv_add (the halo
    exchange excluded, like the reference's per_partition_ns).  Failed
    conversions are skipped; both parts are restored to CSR at the end.
    Returns {"entries": {(lf, rf): seconds}, "skipped": [...],
    "convert_s": {(lf, rf): seconds}}."""
    import statistics
    import time

    import torch
    from .datamove import convert_inplace
    from .errors import DynSparseError
    from .formats import FormatId
    from .kernels import prepared_spmv, spmv, spmv_add, SERIAL
    from .tuner import FORMATS
    dev = split.local.device
    n = part.a_full.nrows
    g = part.halo.ghost_count
    remote_axis = FORMATS if g > 0 else (FormatId.CSR,)
    x = DenseVector.ones(n + g, MemorySpace.DEVICE, dev)
    y = DenseVector.zeros(n, MemorySpace.DEVICE, dev)
    xo, xg = DenseVector(x.data[:n]), DenseVector(x.data[n:])
    entries, skipped, conv = {}, [], {}
    for lf in FORMATS:
        for rf in remote_axis:
            try:   # once untimed: fill-limit check, and the memory pool grows here
                convert_inplace(split.local, lf, fill_limit)
                convert_inplace(split.remote, rf, fill_limit)
            except DynSparseError:
                skipped.append((lf, rf))
                convert_inplace(split.local, FormatId.CSR)
                convert_inplace(split.remote, FormatId.CSR)
                continue
            convert_inplace(split.local, FormatId.CSR)
            convert_inplace(split.remote, FormatId.CSR)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()   # the switching cost proper (warm pool)
            convert_inplace(split.local, lf, fill_limit)
            convert_inplace(split.remote, rf, fill_limit)
            torch.cuda.synchronize(dev)
            conv[(lf, rf)] = time.perf_counter() - t0
            st = torch.cuda.current_stream(dev)
            spmv(SERIAL, split.local, xo, y)          # warm-up, untimed
            spmv_add(SERIAL, split.remote, xg, y)
            # the events must bracket device work: launchers prepared up front
            # (descriptors, plans), so each rep costs two ctypes calls of host time
            lo = prepared_spmv(split.local, xo, y, 0)
            ro = prepared_spmv(split.remote, xg, y, 1)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(reps)]
            for a, b in ev:
                a.record(st)
                lo()
                ro()
                b.record(st)
            torch.cuda.synchronize(dev)
            med = statistics.median(a.elapsed_time(b) for a, b in ev) * 1e-3
            entries[(lf, rf)] = max(med, 1e-9)
            convert_inplace(split.local, FormatId.CSR)
            convert_inplace(split.remote, FormatId.CSR)
    if g == 0:   # no ghosts: the remote format cannot matter (tuner.py:112-118)
        for (lf, _), t in list(entries.items()):
            for rf in FORMATS:
                entries[(lf, rf)] = t
    return {"entries": entries, "skipped": skipped, "convert_s": conv}


def select_rank_plan(entries: dict, mode: str = "multi", world: int = 1):
    """(local, remote) for THIS rank (tuner.py:146-180): ``multi`` is the
    rank-local argmin (ties to the lower FormatId, local first); ``morpheus``
    / ``ghost`` pick one format for all ranks minimising the max over ranks
    (all-reduce MAX across processes)."""
    from .errors import EmptySearchSpace
    from .formats import FormatId
    from .tuner import FORMATS
    if mode == "fixed":
        return (FormatId.CSR, FormatId.CSR)
    if mode == "multi":
        cands = [(t, lf, rf) for (lf, rf), t in entries.items()]
        if not cands:
            raise EmptySearchSpace("this partition has no measured combination")
        _, lf, rf = min(cands)
        return (lf, rf)
    if mode not in ("morpheus", "ghost"):
        raise ValueError(f"unknown mode {mode!r}")
    import torch
    vary_local = mode == "morpheus"
    vals = []
    for f in FORMATS:
        cell = (f, FormatId.CSR) if vary_local else (FormatId.CSR, f)
        vals.append(entries.get(cell, float("inf")))
    t = torch.tensor(vals, dtype=torch.float64)
    if world > 1:
        import torch.distributed as dist
        t = t.cuda() if dist.get_backend() == "nccl" else t
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    worst = t.cpu().tolist()
    best = min(range(len(FORMATS)), key=lambda i: (worst[i], i))
    if worst[best] == float("inf"):
        raise EmptySearchSpace("no format was measured on every partition")
    f = FORMATS[best]
    return (f, FormatId.CSR) if vary_local else (FormatId.CSR, f)


__all__ = ["HaloSchedule", "RankCG", "init_comm", "rank_cg", "profile_rank", "select_rank_plan",
           "MemorySpace"]
