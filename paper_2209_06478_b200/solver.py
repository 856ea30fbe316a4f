"""Unpreconditioned CG on the device (solver.py:1-234 of the reference).

The recurrence is the reference's, operation for operation (solver.py:73-189):

    r = 1*b + (-1)*(A x0);  ||b||;  rr = r.r;  history[0] = sqrt(rr)/scale
    p = 1*r + 0*r
    repeat:  Ap = A p;  pAp = p.Ap  (breakdown iff pAp <= 0);  alpha = rr/pAp
             x = 1*x + alpha*p;  r = 1*r + (-alpha)*Ap;  rr' = r.r
             history += sqrt(rr')/scale;  stop iff <= tol
             p = 1*r + (rr'/rr)*p

but every scalar lives on the device (ds_cg_scalars): the fused kernels
compute p.Ap inside the SpMV epilogue and r.r inside the x/r update, and the
block that completes a reduction also derives alpha / beta / history /
convergence.  Once ``done`` is set every later kernel is a no-op, so the
host enqueues whole chunks of iterations (optionally as one CUDA graph) and
reads 80 bytes back per chunk; iteration counts and histories stay exact.

Distributed problems (DistributedOperator) run all partitions from this one
controller like the reference (partition dots summed in rank order by the
finalize kernel); dist.py runs one partition per process over NCCL.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import BreakdownZeroCurvature, DimensionMismatch, ValidationFailed
from .formats import DenseVector, DynamicMatrix, FormatId, MemorySpace
from .kernels import ExecBackend, descriptor, extract_diagonal, update_diagonal
from .stencil import PartitionedProblem, SplitMatrix, device_halo, distributed_spmv

PAP, RR = _native.DS_CG_STAGE_PAP, _native.DS_CG_STAGE_RR
DEFERRED = _native.DS_CG_STAGE_DEFERRED


@dataclass
class CgResult:
    """x, iterations, relative residual history (iterations + 1 entries),
    converged (solver.py:23-34)."""

    x: DenseVector | list[DenseVector]
    iterations: int
    residual_history: np.ndarray
    converged: bool


@dataclass
class DistributedOperator:
    problem: PartitionedProblem
    splits: list[SplitMatrix]


@dataclass
class ValidationReport:
    passed: bool
    converged: bool
    iterations: int
    iteration_bound: int
    final_residual: float


# ---------------------------------------------------------------------------
# device CG engine
# ---------------------------------------------------------------------------

class _Part:
    """One partition's device state."""

    def __init__(self, local, remote, n, ghosts, device):
        import torch
        self.local, self.remote, self.n = local, remote, n
        self.d_local = descriptor(local)
        # an EMPTY remote part only turns y into y + 0.0 (kernels.py:196-198):
        # fold that into the local kernel's epilogue instead of a second pass
        self.fold_remote = (remote is not None and remote.nnz == 0
                            and not os.environ.get("DS_NO_FOLD"))
        self.d_remote = descriptor(remote) if remote is not None and not self.fold_remote else None
        self.local_mode = 2 if self.fold_remote else 0
        f64 = dict(dtype=torch.float64, device=device)
        # one allocation for the iteration's vectors (p with its ghost slots,
        # x, r, Ap), each segment 256-B aligned: one persisting-L2 window
        # covers them all (CgEngine._capture)
        seg = lambda m: (m + 31) // 32 * 32   # noqa: E731  (doubles, 256-B multiple)
        sizes = [seg(n + ghosts), seg(n), seg(n), seg(n)]
        self.vec_block = torch.zeros(sum(sizes), **f64)
        offs = [0]
        for z in sizes[:-1]:
            offs.append(offs[-1] + z)
        self.p_full = self.vec_block[offs[0]:offs[0] + n + ghosts]
        self.p = self.p_full[:n]
        self.x = self.vec_block[offs[1]:offs[1] + n]
        self.r = self.vec_block[offs[2]:offs[2] + n]
        self.ap = self.vec_block[offs[3]:offs[3] + n]
        self.b = None
        self.halo = []   # (src partition, count, idx tensor, dst offset in p_full)


class CgEngine:
    """Device-resident CG over one or more partitions on one device."""

    def __init__(self, parts: list[_Part], device, tol: float, max_iters: int):
        import torch
        from . import _device
        self.parts, self.dev = parts, device
        self.tol, self.max_iters = float(tol), int(max_iters)
        self.P = len(parts)
        f64 = dict(dtype=torch.float64, device=device)
        self.scal = torch.zeros(_native.CG_SCALARS_BYTES // 8, **f64)
        self.hist = torch.zeros(max(self.max_iters, 0) + 1, **f64)
        # [bb(P) | rr0(P) | pap(P) | rr(P)] partition partial dots
        self.dots = torch.zeros(4 * self.P, **f64)
        self.lib = _native.load()
        self.ws = _device.workspace(device)
        self.graph = None

    # pointers ---------------------------------------------------------------
    def _p(self, t):
        return t.data_ptr()

    def _dot(self, which: int, k: int) -> int:
        return self.dots.data_ptr() + 8 * (which * self.P + k)

    def _ck(self, rc):
        _native.check(rc)

    # setup (solver.py:88-101 / 147-167) --------------------------------------
    def setup(self, stream) -> None:
        lib, s = self.lib, self._p(self.scal)
        self._exchange(stream, guard=None)
        # x0 = 0 with a DIA operator and no remote part: A x0 is +0.0 in
        # every row (the DIA sum starts from +0.0 and adds +-0.0 products),
        # so Ap is cleared instead of running the SpMV -- bitwise the same
        skip = (getattr(self, "x0_zero", False) and self.P == 1
                and self.parts[0].d_remote is None
                and self.parts[0].d_local.format == int(FormatId.DIA))
        for k, pt in enumerate(self.parts):
            if skip:
                import torch
                with torch.cuda.stream(torch.cuda.ExternalStream(stream, device=self.dev)):
                    pt.ap.zero_()
            else:
                self._ck(lib.ds_cg_spmv_dot(ctypes.byref(pt.d_local), self._p(pt.p_full),
                                            self._p(pt.ap), pt.local_mode, None, None, 0, None,
                                            None, None, 0, self._p(self.ws), stream))
            if pt.d_remote is not None:
                self._ck(lib.ds_cg_spmv_dot(ctypes.byref(pt.d_remote),
                                            self._p(pt.p_full) + 8 * pt.n, self._p(pt.ap), 1,
                                            None, None, 0, None, None, None, 0,
                                            self._p(self.ws), stream))
            self._ck(lib.ds_cg_setup_residual(pt.n, self._p(pt.b), self._p(pt.ap),
                                              self._p(pt.r), self._p(pt.p), self._dot(0, k),
                                              self._dot(1, k), self._p(self.ws), stream))
        self._ck(lib.ds_cg_setup_finalize(s, self._dot(0, 0), self._dot(1, 0), self.P, self.tol,
                                          self.max_iters, self._p(self.hist), stream))

    def _exchange(self, stream, guard) -> None:
        for pt in self.parts:
            for q, cnt, idx, off in pt.halo:
                self._ck(self.lib.ds_cg_gather(cnt, self._p(idx), self._p(self.parts[q].p_full),
                                               self._p(pt.p_full) + 8 * off, guard, stream))

    # one iteration (solver.py:102-116 / 170-188) ------------------------------
    def step(self, stream) -> None:
        lib, s, hist = self.lib, self._p(self.scal), self._p(self.hist)
        P, ws = self.P, self._p(self.ws)
        if P == 1 and self.parts[0].d_remote is None and not os.environ.get("DS_CG_TICKETS"):
            return self._step_deferred(stream)
        fin = 1 if P == 1 else 0
        self._exchange(stream, guard=s)
        marks = getattr(self, "_marks", None)
        for k, pt in enumerate(self.parts):
            if marks is not None and k == 0:
                marks[1].record(marks[0])
            if pt.d_remote is None:
                self._ck(lib.ds_cg_spmv_dot(ctypes.byref(pt.d_local), self._p(pt.p_full),
                                            self._p(pt.ap), pt.local_mode, self._p(pt.p),
                                            self._dot(2, k),
                                            PAP, s, hist, self._dot(2, 0), fin, ws, stream))
            else:
                self._ck(lib.ds_cg_spmv_dot(ctypes.byref(pt.d_local), self._p(pt.p_full),
                                            self._p(pt.ap), 0, None, None, 0, s, None, None, 0,
                                            ws, stream))
                if marks is not None and k == 0:
                    marks[2].record(marks[0])
                    marks = None
                self._ck(lib.ds_cg_spmv_dot(ctypes.byref(pt.d_remote),
                                            self._p(pt.p_full) + 8 * pt.n, self._p(pt.ap), 1,
                                            self._p(pt.p), self._dot(2, k), PAP, s, hist,
                                            self._dot(2, 0), fin, ws, stream))
            if marks is not None and k == 0:
                marks[2].record(marks[0])
                marks = None
        if not fin:
            self._ck(lib.ds_cg_finalize(PAP, s, hist, self._dot(2, 0), P, stream))
        for k, pt in enumerate(self.parts):
            self._ck(lib.ds_cg_update(pt.n, self._p(pt.x), self._p(pt.r), self._p(pt.p),
                                      self._p(pt.ap), s, self._dot(3, k), hist,
                                      self._dot(3, 0), fin, ws, stream))
        if not fin:
            self._ck(lib.ds_cg_finalize(RR, s, hist, self._dot(3, 0), P, stream))
        for pt in self.parts:
            self._ck(lib.ds_cg_direction(pt.n, self._p(pt.r), self._p(pt.p), s, stream))

    def _step_deferred(self, stream) -> None:
        """Single partition: 3 kernels, no reduction tails -- the SpMV and the
        update leave fixed-order block partials that the next kernel reduces
        (DS_CG_STAGE_DEFERRED)."""
        lib, s, hist, ws = self.lib, self._p(self.scal), self._p(self.hist), self._p(self.ws)
        pt = self.parts[0]
        marks = getattr(self, "_marks", None)
        if marks is not None:
            marks[1].record(marks[0])
        self._ck(lib.ds_cg_spmv_dot(ctypes.byref(pt.d_local), self._p(pt.p_full),
                                    self._p(pt.ap), pt.local_mode, self._p(pt.p), self._dot(2, 0),
                                    DEFERRED, s, hist, None, 0, ws, stream))
        if marks is not None:
            marks[2].record(marks[0])
        if not os.environ.get("DS_CG_UNFUSED"):
            rc = lib.ds_cg_update_direction_deferred(pt.n, self._p(pt.x), self._p(pt.r),
                                                     self._p(pt.p), self._p(pt.ap), s, hist, ws,
                                                     stream)
            if rc != _native.DS_ERR_NOT_SUPPORTED:
                self._ck(rc)
                self._tail_launches = 1
                return
        self._tail_launches = 2
        self._ck(lib.ds_cg_update_deferred(pt.n, self._p(pt.x), self._p(pt.r), self._p(pt.p),
                                           self._p(pt.ap), s, ws, stream))
        self._ck(lib.ds_cg_direction_deferred(pt.n, self._p(pt.r), self._p(pt.p), s, hist, ws,
                                              stream))

    def scalars(self) -> _native.DsCgScalars:
        raw = self.scal.cpu().numpy().tobytes()
        return _native.DsCgScalars.from_buffer_copy(raw)

    def run(self, chunk: int | None = None, use_graph: bool | None = None) -> _native.DsCgScalars:
        """Enqueue iterations in chunks until ``done`` (one 80-byte readback per chunk)."""
        import torch
        from . import _device
        dev = self.dev
        with torch.cuda.device(dev):
            st = _device.stream(dev)
            self.setup(st)
            if use_graph is None:
                use_graph = self.max_iters >= 16
            # the whole loop on the device (one graph launch, one readback);
            # no readback first: a solve that setup already finished (b = 0,
            # max_iters = 0) makes every step a no-op
            if use_graph and _WHILE_STEPS > 0 and getattr(self, "_while", None) is not False:
                if getattr(self, "_while", None) is None:
                    self._capture_while(_WHILE_STEPS)
                else:
                    self._persist_on(st)
                if self._while:
                    try:
                        _native.check(self.lib.ds_graph_exec_launch(self._while[1], st))
                        return self.scalars()
                    finally:
                        self.release_l2(st)
            sc = self.scalars()
            if sc.done:
                return sc
            c = chunk or (8 if use_graph else 4)
            if use_graph and self.graph is None:
                self._capture(c)
            elif use_graph:
                self._persist_on(st)
            try:
                return self._run_rounds(c, use_graph, st)
            finally:
                self.release_l2(st)

    def _run_rounds(self, c: int, use_graph: bool, st) -> _native.DsCgScalars:
        rounds = 1
        while True:
            # replays between readbacks grow geometrically (1, 1, 2, 4, ...
            # graphs of c steps): after convergence every kernel is a
            # no-op, so overshooting costs only launch latency
            for _ in range(rounds):
                if use_graph:
                    self.graph.replay()
                else:
                    for _ in range(c):
                        self.step(st)
            sc = self.scalars()
            if sc.done:
                return sc
            rounds = min(rounds * 2, _MAX_ROUNDS)

    def _capture_while(self, k: int) -> None:
        """Capture the solve loop as ONE graph: a WHILE conditional node whose
        body is ``k`` iterations + the continue kernel (condition = not
        done).  Sets self._while = (graph, exec, workspace) or False when the
        driver refuses (the chunked replays are used then)."""
        import torch
        from . import _device
        cap = torch.cuda.Stream(self.dev)
        cap.wait_stream(torch.cuda.current_stream(self.dev))
        ws = _device.new_workspace(self.dev)   # owned by this graph
        torch.cuda.synchronize(self.dev)
        saved, self.ws = self.ws, ws
        if self.P == 1 and os.environ.get("DS_CG_L2_PERSIST", "1") != "0":
            vb = self.parts[0].vec_block
            self._l2_persist = self.lib.ds_l2_persist(vb.data_ptr(), vb.numel() * 8,
                                                      cap.cuda_stream) == 0
        g, h, ex = ctypes.c_void_p(), ctypes.c_ulonglong(), ctypes.c_void_p()
        self._while = False
        if self.lib.ds_while_graph_begin(cap.cuda_stream, ctypes.byref(g), ctypes.byref(h)):
            self.ws = saved
            return
        rc = 0
        try:
            for _ in range(k):
                self.step(cap.cuda_stream)
            rc = self.lib.ds_cg_while_continue(h.value, self._p(self.scal), cap.cuda_stream)
        finally:
            rc = self.lib.ds_while_graph_end(cap.cuda_stream, g, ctypes.byref(ex)) or rc
            self.ws = saved
        if rc:
            self.lib.ds_graph_destroy(g, ex)
            return
        self._while = (g.value, ex.value, ws)

    def __del__(self):
        w = getattr(self, "_while", None)
        if w:
            try:
                self.lib.ds_graph_destroy(w[0], w[1])
            except Exception:  # pragma: no cover - interpreter shutdown
                pass

    def _persist_on(self, stream) -> None:
        """Re-establish the persisting-L2 carve-out for a replay of a graph
        captured with the vectors' window (the window lives in the graph's
        kernel nodes, but release_l2 gave the carve-out back after the last
        solve: without it the window persists nothing; WHILE loop at 104^3
        8.27 -> 8.17 ms, A/B on one box, DS_CG_REPERSIST=0 to compare)."""
        if (self.P == 1 and os.environ.get("DS_CG_L2_PERSIST", "1") != "0"
                and os.environ.get("DS_CG_REPERSIST", "1") != "0"):
            vb = self.parts[0].vec_block
            self._l2_persist = self.lib.ds_l2_persist(vb.data_ptr(), vb.numel() * 8,
                                                      stream) == 0

    def release_l2(self, stream) -> None:
        """Give the persisting-L2 carve-out back (set by _capture)."""
        if getattr(self, "_l2_persist", False):
            self.lib.ds_l2_persist_reset(stream)
            self._l2_persist = False

    # benchmarking hooks ---------------------------------------------------
    def capture_step(self, steps: int = 1) -> None:
        """Capture ``steps`` iterations as one CUDA graph (replayed by ``replay``)."""
        self._capture(steps)

    def replay(self) -> None:
        self.graph.replay()

    def launches_per_step(self) -> int:
        if getattr(self, "_tail_launches", None) is not None:   # deferred single-partition step
            return 1 + self._tail_launches
        n = sum(1 for pt in self.parts for h in pt.halo if h[1])
        for pt in self.parts:
            n += 1 + (pt.d_remote is not None) + 2      # spmv(s), update, direction
        return n + (2 if self.P > 1 else 0)              # finalize kernels

    def time_spmv_in_steps(self, steps: int, stream_handle=None) -> dict:
        """Eager iterations with CUDA events around partition 0's local SpMV
        launch (the dominant kernel) and around each whole step."""
        import torch
        st = torch.cuda.current_stream(self.dev)
        lib, ws = self.lib, self._p(self.ws)
        ev = []
        for _ in range(steps):
            a, b, c, d = (torch.cuda.Event(enable_timing=True) for _ in range(4))
            a.record(st)
            self._step_with_marks(st, b, c)
            d.record(st)
            ev.append((a, b, c, d))
        torch.cuda.synchronize(self.dev)
        k = [b.elapsed_time(c) for _, b, c, _ in ev]
        s = [a.elapsed_time(d) for a, _, _, d in ev]
        del lib, ws
        return {"avg_ms": sum(k) / len(k), "step_ms": sum(s) / len(s), "launches": len(k)}

    def time_spmv_in_graph(self, steps: int, per_graph: int = 10) -> dict | None:
        """The dominant kernel's duration inside graph-replayed steps, as the
        bench runs them: ``per_graph`` steps captured in one graph (with the
        vectors' persisting-L2 window, like ``capture_step``) with external
        timing events around every step's local SpMV node and around the
        whole graph, replayed until ``steps`` SpMVs were timed.  The events
        are recorded by the device at the node boundaries (no host latency);
        they do stand between the tail and the next SpMV, so the SpMV's
        programmatic early start is not counted in its favour.  None if this
        torch cannot capture timing events."""
        import torch
        from . import _device
        cap = torch.cuda.Stream(self.dev)
        cap.wait_stream(torch.cuda.current_stream(self.dev))
        ws = _device.new_workspace(self.dev)   # owned by this graph (kept on the engine)
        torch.cuda.synchronize(self.dev)
        try:
            a, d = (torch.cuda.Event(enable_timing=True, external=True) for _ in range(2))
            marks = [(torch.cuda.Event(enable_timing=True, external=True),
                      torch.cuda.Event(enable_timing=True, external=True))
                     for _ in range(per_graph)]
        except TypeError:
            return None
        persist = False
        if self.P == 1 and os.environ.get("DS_CG_L2_PERSIST", "1") != "0":
            vb = self.parts[0].vec_block
            persist = self.lib.ds_l2_persist(vb.data_ptr(), vb.numel() * 8, cap.cuda_stream) == 0
        saved, self.ws = self.ws, ws
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g, stream=cap):
                a.record(cap)
                for b, c in marks:
                    self._marks = (cap, b, c)
                    try:
                        self.step(cap.cuda_stream)
                    finally:
                        self._marks = None
                d.record(cap)
        finally:
            self.ws = saved
        k, s = [], []
        for _ in range(max(1, steps // per_graph)):
            g.replay()
            torch.cuda.synchronize(self.dev)
            k.extend(b.elapsed_time(c) for b, c in marks)
            s.append(a.elapsed_time(d) / per_graph)
        if persist:
            self.lib.ds_l2_persist_reset(cap.cuda_stream)
        return {"avg_ms": sum(k) / len(k), "step_ms": sum(s) / len(s), "launches": len(k),
                "method": f"graphs of {per_graph} steps (the bench's), external timing events "
                          f"around every SpMV node"}

    def _step_with_marks(self, st, mark0, mark1) -> None:
        self._marks = (st, mark0, mark1)
        try:
            self.step(st.cuda_stream)
        finally:
            self._marks = None

    def _capture(self, c: int) -> None:
        import torch
        from . import _device
        cap = torch.cuda.Stream(self.dev)
        cap.wait_stream(torch.cuda.current_stream(self.dev))
        ws = _device.new_workspace(self.dev)   # owned by this graph (kept on the engine)
        torch.cuda.synchronize(self.dev)
        saved, self.ws = self.ws, ws
        # keep the vectors L2-resident across iterations (captured into the
        # graph's kernel nodes); the matrix streams with evict_first
        persist = (self.P == 1 and os.environ.get("DS_CG_L2_PERSIST", "1") != "0")
        if persist:
            vb = self.parts[0].vec_block
            persist = self.lib.ds_l2_persist(vb.data_ptr(), vb.numel() * 8,
                                             cap.cuda_stream) == 0
            self._l2_persist = persist
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g, stream=cap):
                st = cap.cuda_stream
                for _ in range(c):
                    self.step(st)
        finally:
            self.ws = saved
        # the window now lives in the graph's kernel nodes; the carve-out
        # (cudaLimitPersistingL2CacheSize) stays set for the replays
        self.graph = g
        self._graph_ws = ws


# graph replays between two scalar readbacks at most (each replay = chunk
# iterations): converged iterations still launch (as no-ops), so the cap
# bounds that overshoot against the cost of a readback
_MAX_ROUNDS = max(1, int(os.environ.get("DS_CG_MAX_ROUNDS", "4")))
# iterations per body of the device-side WHILE loop (0: chunked replays)
_WHILE_STEPS = max(0, int(os.environ.get("DS_CG_WHILE_STEPS", "8")))   # e2e solve: 4 -> 1068 vs 16 -> 994 GFLOP/s


def _finish(engine: CgEngine, sc) -> tuple[int, np.ndarray, bool]:
    it = int(sc.iter)
    if sc.done == 2:
        raise BreakdownZeroCurvature(f"p'Ap = {sc.pap} at iteration {it + 1}")
    hist = engine.hist[:it + 1].cpu().numpy().copy()
    return it, hist, sc.done == 1


# ---------------------------------------------------------------------------
# public API
# ---------------------------------------------------------------------------

def cg(backend: ExecBackend, a, b, x0=None, tol: float = 1e-9, max_iters: int = 500,
       use_graph: bool | None = None) -> CgResult:
    """CG for SPD systems (solver.py:56-70): ``a`` is a container, a
    DynamicMatrix or a DistributedOperator (then b / x0 are per-partition
    owned vectors).  Stops when ||r||/||b|| <= tol or after max_iters; raises
    BreakdownZeroCurvature when p'Ap <= 0."""
    if tol <= 0:
        raise ValueError(f"tol must be positive, got {tol}")
    if isinstance(a, DistributedOperator):
        return _cg_distributed(a, b, x0, tol, max_iters, use_graph)
    return _cg_single(a, b, x0, tol, max_iters, use_graph)


def _cg_single(a, b, x0, tol, max_iters, use_graph):
    import torch
    from .datamove import to_device
    from .kernels import _exec_device
    mat = a.payload if isinstance(a, DynamicMatrix) else a
    if mat.nrows != mat.ncols:
        raise DimensionMismatch(f"cg needs a square matrix, got {mat.nrows}x{mat.ncols}")
    n = mat.nrows
    if b.length != n:
        raise DimensionMismatch(f"b length {b.length} != {n}")
    if x0 is not None and x0.length != n:
        raise DimensionMismatch(f"x0 length {x0.length} != {n}")
    dev = _exec_device(mat, b, x0)
    A = to_device(mat, dev)
    with torch.cuda.device(dev):
        pt = _Part(A, None, n, 0, dev)
        pt.b = to_device(b, dev).data
        if x0 is not None:
            pt.p_full.copy_(to_device(x0, dev).data)   # setup computes A x0 from p_full
            pt.x.copy_(pt.p_full)
        eng = CgEngine([pt], dev, tol, max_iters)
        eng.x0_zero = x0 is None
        sc = eng.run(use_graph=use_graph)
        it, hist, conv = _finish(eng, sc)
        x = DenseVector(pt.x)
    if b.space == MemorySpace.HOST:
        x = DenseVector(pt.x.cpu().numpy())
    return CgResult(x, it, hist, conv)


def build_engine(op: DistributedOperator, bs, x0s, tol, max_iters) -> tuple[CgEngine, list]:
    """Device engine for a single-controller DistributedOperator."""
    import torch
    from .datamove import to_device
    from .kernels import _exec_device
    problem, splits = op.problem, op.splits
    P = problem.npartitions
    n = problem.spec.local_points
    if len(bs) != P:
        raise DimensionMismatch(f"expected {P} right-hand sides, got {len(bs)}")
    for v in bs:
        if v.length != n:
            raise DimensionMismatch(f"b length {v.length} != local size {n}")
    if x0s is not None:
        if len(x0s) != P:
            raise DimensionMismatch(f"expected {P} initial guesses, got {len(x0s)}")
        for v in x0s:
            if v.length != n:
                raise DimensionMismatch(f"x0 length {v.length} != local size {n}")
    dev = _exec_device(splits[0].local.payload, *bs)
    parts = []
    with torch.cuda.device(dev):
        for k, (part, split) in enumerate(zip(problem.partitions, splits)):
            loc = to_device(split.local.payload, dev)
            rem = to_device(split.remote.payload, dev)
            pt = _Part(loc, rem, n, part.halo.ghost_count, dev)
            pt.b = to_device(bs[k], dev).data
            if x0s is not None:
                pt.x.copy_(to_device(x0s[k], dev).data)
                pt.p.copy_(pt.x)
            # recv starts are absolute slots (n + ghost index) into p_full
            pt.halo = [(q, cnt, idx, start)
                       for q, cnt, idx, start in device_halo(part, dev) if cnt]
            parts.append(pt)
    return CgEngine(parts, dev, tol, max_iters), parts


def _pinned(eng, name: str, n: int):
    """Pinned host staging buffer cached on the engine (allocated once)."""
    import torch
    buf = eng.__dict__.setdefault("_pins", {}).get((name, n))
    if buf is None:
        buf = torch.empty(n, dtype=torch.float64, pin_memory=True)
        eng._pins[(name, n)] = buf
    return buf


def _pinned_result(eng, k: int, n: int):
    """A pinned host buffer for a result array handed to the caller: a pool
    per partition on the engine; an entry is reused only once every numpy
    array (or view) over it has been released -- the numpy arrays reference a
    ctypes view of the buffer, whose reference count tells.  The ctypes view
    keeps the pinned tensor alive, so a returned array outlives the engine."""
    import sys
    import torch
    pool = eng.__dict__.setdefault("_xpool", {}).setdefault((k, n), [])
    for ent in pool:
        if sys.getrefcount(ent[1]) == 2:   # only the pool entry and the argument
            return ent
    t = torch.empty(n, dtype=torch.float64, pin_memory=True)
    c = (ctypes.c_double * n).from_address(t.data_ptr())
    c._keep = t
    ent = (t, c)
    pool.append(ent)
    return ent


def _pinned_copy(eng, name: str, dst, src_np) -> None:
    """Host numpy -> device tensor through a cached pinned staging buffer
    (DS_PAGEABLE_STAGING=1: a direct pageable copy -- faster in a fresh
    process, 1.6x slower inside bench.py's, so not the default)."""
    import torch
    if os.environ.get("DS_PAGEABLE_STAGING"):
        dst.copy_(torch.from_numpy(np.ascontiguousarray(src_np)))
        return
    buf = _pinned(eng, name, dst.numel())
    main = torch.cuda.current_stream(dst.device)
    main.synchronize()   # buffer free for reuse
    src = torch.from_numpy(np.ascontiguousarray(src_np))
    # in 4 pieces: the DMA of a piece overlaps the host copy of the next, and
    # the pieces alternate between two streams (two copy engines: a 9 MB H2D
    # 0.25 -> 0.19 ms, tools/h2d_probe2.py)
    side = eng.__dict__.get("_h2d_side")
    if side is None:
        side = eng._h2d_side = torch.cuda.Stream(dst.device)
    side.wait_stream(main)
    n = dst.numel()
    step = max(1 << 16, -(-n // 4))
    for i, a in enumerate(range(0, n, step)):
        b = min(n, a + step)
        buf[a:b].copy_(src[a:b])   # multi-threaded host copy
        with torch.cuda.stream(side if i % 2 else main):
            dst[a:b].copy_(buf[a:b], non_blocking=True)
    main.wait_stream(side)


def _reload(eng: CgEngine, bs, x0s) -> None:
    """Refill a cached engine's right-hand sides / initial guesses in place
    (its captured graph keeps pointing at the same buffers)."""
    for k, pt in enumerate(eng.parts):
        src = bs[k]
        if src.space == MemorySpace.HOST:
            _pinned_copy(eng, f"b{k}", pt.b, src.data)
        else:
            pt.b.copy_(src.data)
        if x0s is None:
            pt.p_full.zero_()     # x0 = 0: x and p (with its ghost slots) zero
            pt.x.zero_()
            continue
        if x0s[k].space == MemorySpace.HOST:
            _pinned_copy(eng, f"x0{k}", pt.x, x0s[k].data)
        else:
            pt.x.copy_(x0s[k].data)
        pt.p.copy_(pt.x)
        pt.p_full[pt.n:].zero_()
    eng.x0_zero = x0s is None


def _cg_distributed(op, bs, x0s, tol, max_iters, use_graph):
    import torch
    # Reuse the engine (device buffers + captured CUDA graph) across calls on
    # the same operator with the same controls -- the analysis-reuse pattern
    # of sparse solvers; a changed matrix format/storage rebuilds it.
    key = (float(tol), int(max_iters), use_graph,
           tuple((sp.local.active, id(sp.local.payload), sp.remote.active, id(sp.remote.payload))
                 for sp in op.splits))
    cached = op.__dict__.get("_cg_engine")
    if cached is not None and cached[0] == key and len(bs) == cached[1].P:
        eng = cached[1]
        _reload(eng, bs, x0s)
    else:
        eng, _ = build_engine(op, bs, x0s, tol, max_iters)
        eng.x0_zero = x0s is None   # fresh vectors are zero
        op.__dict__["_cg_engine"] = (key, eng)
    parts = eng.parts
    with torch.cuda.device(eng.dev):
        sc = eng.run(use_graph=use_graph)
        it, hist, conv = _finish(eng, sc)
    host = bs[0].space == MemorySpace.HOST
    if host and not os.environ.get("DS_PAGEABLE_STAGING"):
        # fresh arrays (the reference returns new ones) in pinned memory: the
        # D2H lands in the returned array itself (no host-side copy, no page
        # faults on freshly allocated pages)
        outs = [_pinned_result(eng, k, pt.n) for k, pt in enumerate(parts)]
        for (t, _), pt in zip(outs, parts):
            t.copy_(pt.x, non_blocking=True)
        torch.cuda.synchronize(eng.dev)
        xs = [DenseVector(np.ctypeslib.as_array(c)) for _, c in outs]
    elif host:   # fresh arrays (the reference returns new ones): one D2H each
        xs = [DenseVector(pt.x.cpu().numpy()) for pt in parts]
    else:
        xs = [DenseVector(pt.x.clone()) for pt in parts]
    return CgResult(xs, it, hist, conv)


def validate_solver(backend: ExecBackend, problem: PartitionedProblem,
                    splits: list[SplitMatrix], diag_value: float = 1.0e6, tol: float = 1e-12,
                    max_iters: int = 50, iteration_bound: int = 12) -> ValidationReport:
    """Diagonal-modification check (solver.py:192-234): diagonal := diag_value,
    b := A 1, CG must reach tol within iteration_bound; diagonals restored
    exactly in every case; ValidationFailed carries the report."""
    n = problem.spec.local_points
    saved = [extract_diagonal(sp.local) for sp in splits]
    space = splits[0].local.space
    dev = splits[0].local.device
    new_diag = DenseVector(np.full(n, diag_value)) if space == MemorySpace.HOST else \
        DenseVector.ones(n, MemorySpace.DEVICE, dev)
    if space == MemorySpace.DEVICE:
        new_diag.data.fill_(diag_value)
    try:
        for sp in splits:
            update_diagonal(sp.local, new_diag)
        ones = [DenseVector.ones(n + p.halo.ghost_count, space, dev) for p in problem.partitions]
        bs = [DenseVector.zeros(n, space, dev) for _ in problem.partitions]
        distributed_spmv(backend, problem, splits, ones, bs)
        res = cg(backend, DistributedOperator(problem, splits), bs, tol=tol, max_iters=max_iters)
    finally:
        for sp, d in zip(splits, saved):
            update_diagonal(sp.local, d)
    passed = res.converged and res.iterations <= iteration_bound
    report = ValidationReport(passed=passed, converged=res.converged, iterations=res.iterations,
                              iteration_bound=iteration_bound,
                              final_residual=float(res.residual_history[-1]))
    if not passed:
        raise ValidationFailed(
            f"validation cg took {res.iterations} iterations (bound {iteration_bound}), "
            f"converged={res.converged}", report=report)
    return report

