"""One partition per process: the distributed CG across GPUs.

The reference simulates MPI ranks as list entries in one process
(stencil.py:9-15); on the B200 node each rank is a process driving one GPU.
torch.distributed only bootstraps (it carries the NCCL unique id or the CUDA
IPC handles); the data path is this library's.  Per CG iteration
(solver.py:170-188):

    Ap        local SpMV (owned entries only) while the halo is in flight,
              then the remote spmv_add fused with the partition's p.Ap
    p.Ap      all-gather of the P partition dots, rank-ordered sum on device
    x, r      update + partition r.r; all-gather; history / beta
    p         p = r + beta p

Two transports move the halo and the dots:

* ``peer`` (default): plain loads/stores on CUDA-IPC-mapped peer memory
  (NVLink / NVSwitch).  After its direction update a rank pushes its boundary
  values straight into each neighbour's ghost slots and raises a flag there;
  the neighbour waits on its flags before the remote spmv_add, i.e. behind
  its local SpMV.  A dot all-gather is one 1-block kernel: remote stores of
  the partition dot into every rank's ``all`` row + flags, then a wait on its
  own.  No NCCL launch sits on the iteration's critical path.  Several ranks
  may share one GPU (the IPC mapping then aliases the same HBM), which is how
  the N > 1 engine is tested on a single B200.
* ``nccl``: pack kernels + one NCCL group of send/recv pairs on a side stream
  (overlapped with the local SpMV) and ncclAllGather of the dots.

Everything is stream-ordered with device-side scalars, so one iteration is
captured once as a CUDA graph and replayed.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native
from .formats import DenseVector, FormatId, MemorySpace
from .kernels import descriptor
from .stencil import GridSpec, PartitionData, SplitMatrix, halo_send_lists

PAP, RR = _native.DS_CG_STAGE_PAP, _native.DS_CG_STAGE_RR
_NSTAGES = 4          # all-gather rows: p.Ap, r.r, b.b (setup), r0.r0 (setup)


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

    def recv_start_of(self) -> dict[int, int]:
        """{owner rank: first ghost slot of its block} -- what each neighbour
        needs to push into this rank's ghosts."""
        return {q: s for q, c, s in zip(self.peers, self.recv_counts, self.recv_starts) if c}


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


def _carray(ty, vals):
    return (ty * max(len(vals), 1))(*vals)


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------

class NcclTransport:
    """Halo over NCCL send/recv (side stream, overlapped with the local SpMV),
    dots over ncclAllGather."""

    name = "nccl"

    def __init__(self, eng, comm=None):
        import torch
        from . import _device
        self.eng = eng
        if comm is None:
            comm, _, _ = init_comm(eng.dev)
        self.comm = comm
        sched = eng.sched
        self.nnbr = len(sched.peers)
        self._send_idx = [_device.to_index_tensor(s, eng.dev) for s in sched.send_idx]
        total = sum(int(s.size) for s in sched.send_idx)
        self._send_buf = torch.zeros(max(total, 1), dtype=torch.float64, device=eng.dev)
        bufs, off = [], 0
        for s in sched.send_idx:
            bufs.append(self._send_buf.data_ptr() + 8 * off)
            off += int(s.size)
        self._c_peers = _carray(ctypes.c_int32, sched.peers)
        self._c_scount = _carray(ctypes.c_int64, [int(s.size) for s in sched.send_idx])
        self._c_sidx = _carray(ctypes.c_void_p, [t.data_ptr() if t.numel() else None
                                                 for t in self._send_idx])
        self._c_sbuf = _carray(ctypes.c_void_p, bufs)
        self._c_rcount = _carray(ctypes.c_int64, sched.recv_counts)
        self._c_rstart = _carray(ctypes.c_int64, sched.recv_starts)
        self.side = torch.cuda.Stream(eng.dev)

    def _exchange(self, stream, s_ptr) -> None:
        e = self.eng
        _native.check(e.lib.ds_halo_exchange(self.nnbr, self._c_peers, self._c_scount,
                                             self._c_sidx, self._c_sbuf, self._c_rcount,
                                             self._c_rstart, e.p_full.data_ptr(), s_ptr,
                                             self.comm, stream))

    def halo_setup(self, stream) -> None:
        self._exchange(stream, None)

    def halo_start(self, main) -> None:
        self.side.wait_stream(main)
        self._exchange(self.side.cuda_stream, self.eng.scal.data_ptr())

    def halo_finish(self, main) -> None:
        main.wait_stream(self.side)

    def after_direction(self, stream) -> None:
        pass

    def allgather(self, k: int, stream) -> None:
        e = self.eng
        _native.check(e.lib.ds_allgather_f64(e.mine.data_ptr() + 8 * k,
                                             e.all.data_ptr() + 8 * k * e.P, 1, self.comm, stream))

    def launches(self) -> int:
        return sum(1 for s in self.eng.sched.send_idx if s.size)

    def close(self) -> None:
        if self.comm:
            _native.check(self.eng.lib.ds_nccl_comm_destroy(self.comm))
            self.comm = None


class PeerTransport:
    """Halo and dots with loads/stores on CUDA-IPC-mapped peer memory.

    This rank's exchange block (``xch``, int32 words): the all-gather flags
    [stage][source rank], the halo flags [source rank], the push ticket.
    ``eng.all`` ([stage][rank] doubles) and ``eng.vec_block`` (p with its
    ghosts first) are exported too; every peer's three blocks are mapped."""

    name = "peer"

    def __init__(self, eng, wait: str | None = None):
        import torch
        import torch.distributed as dist
        from . import _device
        self.eng = eng
        lib = eng.lib
        wait = (wait or os.environ.get("DS_PEER_WAIT", "spin")).lower()
        if wait not in ("spin", "memop"):
            raise ValueError(f"DS_PEER_WAIT must be spin or memop, got {wait!r}")
        self.mode = _native.DS_PEER_WAIT_SPIN if wait == "spin" else _native.DS_PEER_WAIT_MEMOP
        P, rank = eng.P, eng.rank
        if P > _native.DS_PEER_MAX_RANKS:
            raise ValueError(f"peer transport handles at most {_native.DS_PEER_MAX_RANKS} ranks")
        self.xch = torch.zeros(_NSTAGES * P + P + 1, dtype=torch.int32, device=eng.dev)
        hb = lib.ds_ipc_handle_bytes()

        def export(t) -> bytes:
            buf = ctypes.create_string_buffer(hb)
            _native.check(lib.ds_ipc_export(t.data_ptr(), buf))
            return buf.raw

        mine = {"vec": export(eng.vec_block), "all": export(eng.all), "xch": export(self.xch),
                "recv_start": eng.sched.recv_start_of()}
        gathered = [None] * P
        torch.cuda.synchronize(eng.dev)
        if P > 1:
            dist.all_gather_object(gathered, mine)
        else:
            gathered = [mine]
        self._opened = []
        vec, allp, xch = [0] * P, [0] * P, [0] * P
        with torch.cuda.device(eng.dev):
            for r, info in enumerate(gathered):
                if r == rank:
                    vec[r], allp[r], xch[r] = (eng.vec_block.data_ptr(), eng.all.data_ptr(),
                                               self.xch.data_ptr())
                    continue
                got = []
                for key in ("vec", "all", "xch"):
                    ptr = ctypes.c_void_p()
                    _native.check(lib.ds_ipc_import(info[key], ctypes.byref(ptr)))
                    self._opened.append(ptr.value)
                    got.append(ptr.value)
                vec[r], allp[r], xch[r] = got
        # all-gather: every rank's all[] and flag rows
        self._c_all = _carray(ctypes.c_void_p, allp)
        self._c_agflag = _carray(ctypes.c_void_p, xch)
        self._my_flags = self.xch.data_ptr()
        # halo push: to each neighbour q this rank sends to, into q's ghost
        # block for this rank, then q's halo flag slot for this rank
        sched = eng.sched
        halo_base = 4 * _NSTAGES * P
        counts, idx, dst, flag = [], [], [], []
        self._send_idx = []
        for q, sidx in zip(sched.peers, sched.send_idx):
            if not sidx.size:
                continue
            start = gathered[q]["recv_start"].get(rank)
            if start is None:
                raise RuntimeError(f"rank {q} has no ghost block for rank {rank}")
            t = _device.to_index_tensor(sidx, eng.dev)
            self._send_idx.append(t)
            counts.append(int(sidx.size))
            idx.append(t.data_ptr())
            dst.append(vec[q] + 8 * int(start))     # p_full sits at the front of vec_block
            flag.append(xch[q] + halo_base + 4 * rank)
        self.nsend = len(counts)
        self._c_counts = _carray(ctypes.c_int64, counts)
        self._c_idx = _carray(ctypes.c_void_p, idx)
        self._c_dst = _carray(ctypes.c_void_p, dst)
        self._c_flag = _carray(ctypes.c_void_p, flag)
        self._ticket = self.xch.data_ptr() + 4 * (_NSTAGES * P + P)
        waits = [self.xch.data_ptr() + halo_base + 4 * q
                 for q, c in zip(sched.peers, sched.recv_counts) if c]
        self.nwait = len(waits)
        self._c_wait = _carray(ctypes.c_void_p, waits)
        if P > 1:
            dist.barrier()     # every mapping is open before anyone writes into it

    def _push(self, stream) -> None:
        e = self.eng
        _native.check(e.lib.ds_peer_halo_push(self.nsend, self._c_counts, self._c_idx,
                                              e.p_full.data_ptr(), self._c_dst, self._c_flag,
                                              self._ticket, stream))

    def _wait(self, stream) -> None:
        _native.check(self.eng.lib.ds_peer_wait_flags(self.nwait, self._c_wait, self.mode,
                                                      stream))

    def halo_setup(self, stream) -> None:
        self._push(stream)
        self._wait(stream)

    def halo_start(self, main) -> None:
        pass      # pushed by the neighbours at the end of their previous step

    def halo_finish(self, main) -> None:
        self._wait(main.cuda_stream)

    def after_direction(self, stream) -> None:
        self._push(stream)

    def allgather(self, k: int, stream) -> None:
        e = self.eng
        _native.check(e.lib.ds_peer_allgather_f64(e.mine.data_ptr() + 8 * k, k, e.rank, e.P,
                                                  self._c_all, self._c_agflag, self._my_flags,
                                                  self.mode, stream))

    def launches(self) -> int:
        spin = self.mode == _native.DS_PEER_WAIT_SPIN
        return (1 if self.nsend else 0) + (1 if self.nwait and spin else 0) + 2

    def close(self) -> None:
        import torch
        if self._opened:
            torch.cuda.synchronize(self.eng.dev)
            for ptr in self._opened:
                self.eng.lib.ds_ipc_close(ptr)
            self._opened = []


# ---------------------------------------------------------------------------
# the engine
# ---------------------------------------------------------------------------

class RankCG:
    """Device CG for this rank's partition; same driver interface as
    solver.CgEngine (setup / step / capture_step / replay / scalars).

    ``transport``: "peer" (default; env DS_TRANSPORT) or "nccl"."""

    def __init__(self, spec: GridSpec, part: PartitionData, split: SplitMatrix, device,
                 tol: float, max_iters: int, comm=None, world: int | None = None,
                 transport: str | None = None):
        import torch
        import torch.distributed as dist
        from . import _device
        from .datamove import to_device
        self.dev = device
        dist_on = dist.is_available() and dist.is_initialized()
        self.P = int(world) if world is not None else (dist.get_world_size() if dist_on else 1)
        self.rank = dist.get_rank() if dist_on else 0
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
        # so one persisting-L2 window covers them (capture_step); p with its
        # ghost slots comes first (the peer transport's push targets)
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
        self.mine = torch.zeros(_NSTAGES, **f64)              # [pap, rr, bb0, rr0] partials
        self.all = torch.zeros(_NSTAGES * self.P, **f64)      # gathered, one row per stage
        self.lib = _native.load()
        self.ws = _device.workspace(device)
        self.sched = HaloSchedule.build(spec, part)
        kind = (transport or os.environ.get("DS_TRANSPORT", "peer")).lower()
        if kind == "peer":
            self.T = PeerTransport(self)
        elif kind == "nccl":
            self.T = NcclTransport(self, comm)
        else:
            raise ValueError(f"unknown transport {kind!r} (peer | nccl)")
        self.graph = None
        self._marks = None

    # -- primitives -----------------------------------------------------------
    def _ck(self, rc):
        _native.check(rc)

    def _allp(self, k):
        return self.all.data_ptr() + 8 * k * self.P

    def _mine(self, k):
        return self.mine.data_ptr() + 8 * k

    # -- CG -------------------------------------------------------------------
    def setup(self, stream) -> None:
        """r = b - A x0 (x0 = the current x, on ``stream`` = torch's current
        stream), p = r, the global b.b / r.r and the first history entry; then
        p's halo for the first iteration (peer transport)."""
        lib, ws = self.lib, self.ws.data_ptr()
        self.p.copy_(self.x)     # the SpMV input of the setup is x0 (solver.py:88-101)
        self.T.halo_setup(stream)
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
        self.T.allgather(2, stream)
        self.T.allgather(3, stream)
        self._ck(lib.ds_cg_setup_finalize(self.scal.data_ptr(), self._allp(2), self._allp(3),
                                          self.P, self.tol, self.max_iters,
                                          self.hist.data_ptr(), stream))
        self.T.after_direction(stream)

    def step(self, stream) -> None:
        """One iteration.  Every kernel no-ops once s->done is set; the
        exchanges themselves always run, so all ranks stay in step."""
        import torch
        lib, ws = self.lib, self.ws.data_ptr()
        s, hist = self.scal.data_ptr(), self.hist.data_ptr()
        main = torch.cuda.ExternalStream(stream, device=self.dev)
        self.T.halo_start(main)
        if self._marks is not None:
            self._marks[1].record(main)
        if self.fold:   # no ghosts: local SpMV + fused partition p.Ap
            self._ck(lib.ds_cg_spmv_dot(ctypes.byref(self.d_local), self.p_full.data_ptr(),
                                        self.ap.data_ptr(), 2, self.p.data_ptr(), self._mine(0),
                                        PAP, s, hist, None, 0, ws, stream))
            if self._marks is not None:
                self._marks[2].record(main)
            self.T.halo_finish(main)
        else:
            self._ck(lib.ds_cg_spmv_dot(ctypes.byref(self.d_local), self.p_full.data_ptr(),
                                        self.ap.data_ptr(), 0, None, None, 0, s, None, None, 0,
                                        ws, stream))
            if self._marks is not None:
                self._marks[2].record(main)
            self.T.halo_finish(main)
            self._ck(lib.ds_cg_spmv_dot(ctypes.byref(self.d_remote),
                                        self.p_full.data_ptr() + 8 * self.n, self.ap.data_ptr(), 1,
                                        self.p.data_ptr(), self._mine(0), PAP, s, hist, None, 0,
                                        ws, stream))
        self.T.allgather(0, stream)
        # alpha from the rank-ordered sum of the gathered p.Ap, x/r update,
        # this partition's r.r -> all-gather -> history / beta / p update
        self._ck(lib.ds_cg_update_gathered(self.n, self.x.data_ptr(), self.r.data_ptr(),
                                           self.p.data_ptr(), self.ap.data_ptr(), s,
                                           self._allp(0), self.P, self._mine(1), ws, stream))
        self.T.allgather(1, stream)
        self._ck(lib.ds_cg_direction_gathered(self.n, self.r.data_ptr(), self.p.data_ptr(), s,
                                              hist, self._allp(1), self.P, ws, stream))
        self.T.after_direction(stream)

    def scalars(self) -> _native.DsCgScalars:
        return _native.DsCgScalars.from_buffer_copy(self.scal.cpu().numpy().tobytes())

    def capture_step(self, steps: int = 1) -> None:
        """Capture ``steps`` iterations (kernels + exchanges) as one CUDA
        graph; fall back to eager launches if capture is refused."""
        import torch
        from . import _device
        cap = torch.cuda.Stream(self.dev)
        ws = _device.new_workspace(self.dev)   # owned by this graph (kept on the engine)
        torch.cuda.synchronize(self.dev)
        saved, self.ws = self.ws, ws
        if os.environ.get("DS_CG_L2_PERSIST", "1") != "0":
            self._l2_persist = self.lib.ds_l2_persist(
                self.vec_block.data_ptr(), self.vec_block.numel() * 8, cap.cuda_stream) == 0
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g, stream=cap):
                for _ in range(steps):
                    self.step(cap.cuda_stream)
            self.graph = g
            self._graph_ws = ws
            self._graph_steps = steps
        except Exception:  # pragma: no cover - depends on the NCCL build / driver
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

    def steps_per_replay(self) -> int:
        return getattr(self, "_graph_steps", 1) if self.graph is not None else 1

    def launches_per_step(self) -> int:
        """This library's kernels per iteration (NCCL's own excluded)."""
        return self.T.launches() + (1 if self.fold else 2) + 2    # + update, direction

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
        """Run to convergence (chunked graph replays) and return this rank's x.
        Every rank reads the same device scalars, so all stop together."""
        import torch
        with torch.cuda.device(self.dev):
            st = torch.cuda.current_stream(self.dev).cuda_stream
            self.setup(st)
            sc = self.scalars()
            if not sc.done:
                if self.graph is None:
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
            self.setup(st.cuda_stream)
            for _ in range(max(1, iters // self.steps_per_replay())):
                self.replay()
            pin[1].copy_(self.x, non_blocking=True)
            st.synchronize()
            return torch.empty_like(pin[1]).copy_(pin[1]).numpy()

    def close(self) -> None:
        if getattr(self, "T", None) is not None:
            self.T.close()
            self.T = None


def rank_cg(spec: GridSpec, part: PartitionData, split: SplitMatrix, tol: float = 1e-9,
            max_iters: int = 500, device=None, transport: str | None = None):
    """CG across processes, one partition per rank (torch.distributed must be
    initialised for more than one rank).  Returns (x_owned DenseVector,
    iterations, history, converged)."""
    from . import _device
    dev = _device.require_cuda(device)
    eng = RankCG(spec, part, split, dev, tol, max_iters, transport=transport)
    try:
        return eng.solve()
    finally:
        eng.close()


# ---------------------------------------------------------------------------
# per-GPU format selection
# ---------------------------------------------------------------------------

def profile_rank(part: PartitionData, split: SplitMatrix, reps: int = 20,
                 fill_limit: int | None = None) -> dict:
    """This rank's row of the tuner's TimingTable (tuner.measure_combination
    per combination; reference tuner.py:53-120).  Returns {"entries":
    {(lf, rf): seconds}, "skipped": [...], "convert_s": {(lf, rf): seconds}}."""
    from .tuner import FORMATS, measure_combination
    dev = split.local.device
    n = part.a_full.nrows
    g = part.halo.ghost_count
    x = DenseVector.ones(n + g, MemorySpace.DEVICE, dev)
    probes = (DenseVector(x.data[:n]), DenseVector(x.data[n:]),
              DenseVector.zeros(n, MemorySpace.DEVICE, dev))
    entries, skipped, conv = {}, [], {}
    for lf in FORMATS:
        for rf in (FORMATS if g > 0 else (FormatId.CSR,)):
            got = measure_combination(split, lf, rf, reps, fill_limit, probes)
            cells = [(lf, rf)] if g > 0 else [(lf, r) for r in FORMATS]
            for cell in cells:
                if got is None:
                    skipped.append(cell)
                else:
                    entries[cell], conv[cell] = got
    return {"entries": entries, "skipped": skipped, "convert_s": conv}


def select_rank_plan(entries: dict, mode: str = "multi", world: int = 1,
                     convert_s: dict | None = None, iterations: int | None = None):
    """(local, remote) for THIS rank (reference tuner.py:146-180 across
    processes): ``multi`` = the rank-local argmin (ties to the lower FormatId,
    local first); ``morpheus`` / ``ghost`` = one format for all ranks, the
    minimum of the max over ranks (all-reduce MAX).  With ``convert_s`` and
    ``iterations`` each cell first pays its switch cost / iterations."""
    from .errors import EmptySearchSpace
    from .tuner import FORMATS, TimingTable, cost_cube, select_plan
    table = TimingTable(entries={(0, lf, rf): t for (lf, rf), t in entries.items()}, reps=1,
                        convert_seconds={(0, lf, rf): t for (lf, rf), t in
                                         (convert_s or {}).items()})
    if mode in ("fixed", "multi"):
        return select_plan(table, mode, iterations).assignments[0]
    if mode not in ("morpheus", "ghost"):
        raise ValueError(f"unknown mode {mode!r}")
    import torch
    cube = cost_cube(table, iterations)[0]
    csr = FORMATS.index(FormatId.CSR)
    side = cube[:, csr] if mode == "morpheus" else cube[csr, :]
    t = torch.tensor(side, dtype=torch.float64)
    if world > 1:
        import torch.distributed as dist
        t = t.cuda() if dist.get_backend() == "nccl" else t
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    worst = t.cpu().numpy()
    if not np.isfinite(worst).any():
        raise EmptySearchSpace("no format was measured on every partition")
    f = FORMATS[int(np.argmin(worst))]
    return (f, FormatId.CSR) if mode == "morpheus" else (FormatId.CSR, f)


__all__ = ["HaloSchedule", "NcclTransport", "PeerTransport", "RankCG", "init_comm", "rank_cg",
           "profile_rank", "select_rank_plan", "MemorySpace"]
