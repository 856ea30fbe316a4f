"""HPCG's multigrid-preconditioned CG on the device.

The reference stops at unpreconditioned CG (solver.py:56-189; SPEC.md:16
lists SymGS/MG as absent), so this module follows the HPCG benchmark that the
paper's Fig. 10 runs: ComputeSYMGS_ref, ComputeMG_ref (3 coarse levels,
restriction of the residual at the even points, injection-style
prolongation) and ComputeCG_ref.  The symmetric Gauss-Seidel sweep is
parallelised with the 8-colour ordering of the 27-point stencil
(colour = x%2 + 2(y%2) + 4(z%2)): rows of one colour never couple, so each
colour is one kernel launch.  Parity: SymGS and the V-cycle are bitwise
identical to the CPU restatement the tests check against (symgs_colored /
mg_vcycle); the PCG residual history matches its pcg_mg within the
dot-product tolerance of the CG tests.  Parity against the reference itself is
UNPINNED -- the reference has no such code.

Single partition (N=1 per process): the coarse-level halo exchanges of a
distributed MG are not built.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import BreakdownZeroCurvature, DimensionMismatch
from .formats import CsrMatrix, DenseVector, FormatId, MemorySpace
from .solver import CgResult
from .stencil import GridSpec, generate_partition

NCOLORS = 8


def stencil_colors(nx: int, ny: int, nz: int) -> np.ndarray:
    """Colour of every local point: x%2 + 2(y%2) + 4(z%2)."""
    i = np.arange(nx * ny * nz, dtype=np.int64)
    return (i % nx) % 2 + 2 * (((i // nx) % ny) % 2) + 4 * ((i // (nx * ny)) % 2)


def _color_lists(colors: np.ndarray):
    """Rows grouped by colour (ascending inside a colour) + colour starts."""
    order = np.argsort(colors, kind="stable").astype(np.int32)
    counts = np.bincount(colors, minlength=NCOLORS).astype(np.int64)
    start = np.zeros(NCOLORS + 1, dtype=np.int64)
    np.cumsum(counts, out=start[1:])
    return order, start


@dataclass
class MgLevel:
    """One grid of the hierarchy: operator, colour lists, the fine-to-coarse
    map to the next level (None on the coarsest) and its work vectors."""

    dims: tuple[int, int, int]
    a: CsrMatrix
    color_rows: object          # int32 device tensor
    color_start: np.ndarray     # int64 host array, NCOLORS + 1
    f2c: object | None          # int32 device tensor (coarse size) or None
    r: object = None
    x: object = None
    axf: object = None
    ell: tuple | None = None    # (width, cols, vals, len, diag) colour-ordered ELL
    oell: tuple | None = None   # (width, host offsets, vals, mask, diag) offset ELL (no columns)
    op: object = None           # the level operator in the SpMV format
    desc: object = None         # cached ds_matrix descriptor of ``op``

    @property
    def nrows(self) -> int:
        return self.a.nrows


@dataclass
class MgHierarchy:
    levels: list[MgLevel] = field(default_factory=list)
    device: object = None

    @staticmethod
    def build(nx: int, ny: int, nz: int, nlevels: int = 4, device=None,
              layout: str = "ell", spmv_format="dia") -> "MgHierarchy":
        """GenerateProblem + GenerateCoarseProblem: each coarse grid halves
        every dimension while all three stay even (at most ``nlevels``).
        ``layout`` "ell" adds the colour-ordered copy the sweep reads
        (coalesced): on levels of >= 2^20 rows the offset ELL (slot q =
        offset q, a presence mask, no column indices: 8 B per slot instead
        of 12; 104^3 sweep 125 -> 110 us) when the off-diagonals fall on <= 32
        offsets, else -- and on the latency-bound coarse levels, where it
        measured slower (35 -> 44 us at 52^3) -- the ELL with columns;
        "oell" / "ell-cols" force one of them; "csr" sweeps the CSR operator
        directly.  The residual
        SpMVs (PCG's A p and the V-cycle's A z) run on the level operator
        converted to ``spmv_format`` -- the runtime format switch applied to
        HPCG (DIA streams the 27 diagonals at ~90% of HBM)."""
        from .datamove import convert
        from .formats import as_format_id
        fmt = as_format_id(spmv_format)
        if layout not in ("ell", "oell", "ell-cols", "csr"):
            raise ValueError(f"layout must be 'ell', 'oell', 'ell-cols' or 'csr', got {layout!r}")
        import torch
        from . import _device
        dev = _device.require_cuda(device)
        h = MgHierarchy(device=dev)
        for lev in range(nlevels):
            part = generate_partition(GridSpec(nx, ny, nz), 0, MemorySpace.DEVICE, dev)
            rows, start = _color_lists(stencil_colors(nx, ny, nz))
            coarsen = lev + 1 < nlevels and nx % 2 == 0 and ny % 2 == 0 and nz % 2 == 0
            f2c = None
            if coarsen:
                cx, cy, cz = nx // 2, ny // 2, nz // 2
                ic = np.arange(cx * cy * cz, dtype=np.int64)
                xc, yc, zc = ic % cx, (ic // cx) % cy, ic // (cx * cy)
                f2c = torch.from_numpy((2 * xc + nx * (2 * yc + ny * 2 * zc))
                                       .astype(np.int32)).to(dev)
            n = nx * ny * nz
            f64 = dict(dtype=torch.float64, device=dev)
            h.levels.append(MgLevel(
                dims=(nx, ny, nz), a=part.a_full, color_rows=torch.from_numpy(rows).to(dev),
                color_start=start, f2c=f2c, r=torch.empty(n, **f64), x=torch.empty(n, **f64),
                axf=torch.empty(n, **f64)))
            if layout == "oell" or (layout == "ell" and n >= _OELL_MIN_ROWS):
                h.levels[-1].oell = _oell(h.levels[-1], dev)
            if layout in ("ell", "oell", "ell-cols") and h.levels[-1].oell is None:
                h.levels[-1].ell = _ell(h.levels[-1], dev)
            h.levels[-1].op = part.a_full if fmt == FormatId.CSR else convert(part.a_full, fmt)
            if not coarsen:
                break
            nx, ny, nz = nx // 2, ny // 2, nz // 2
        return h

    # -- kernels ----------------------------------------------------------
    def _stream(self):
        from . import _device
        return _device.stream(self.device)

    def symgs(self, lev: int, r, x, st=None) -> None:
        """One symmetric colour sweep in place on level ``lev`` (ds_symgs_ell,
        or ds_symgs on the CSR operator)."""
        L = self.levels[lev]
        a = L.a
        cs = L.color_start.ctypes.data_as(_native.P_i64)
        st = self._stream() if st is None else st
        if L.oell is not None:
            w, of, ov, mk, dg = L.oell
            _native.call("ds_symgs_oell", a.nrows, w, of.ctypes.data, L.color_rows.data_ptr(), cs,
                         NCOLORS, ov.data_ptr(), mk.data_ptr(), dg.data_ptr(), r.data_ptr(),
                         x.data_ptr(), st)
            return
        if L.ell is not None:
            w, ec, ev, el, dg = L.ell
            _native.call("ds_symgs_ell", a.nrows, w, L.color_rows.data_ptr(), cs, NCOLORS,
                         ec.data_ptr(), ev.data_ptr(), el.data_ptr(), dg.data_ptr(),
                         r.data_ptr(), x.data_ptr(), st)
            return
        _native.call("ds_symgs", a.nrows, a.row_offsets.data_ptr(), a.col_indices.data_ptr(),
                     a.values.data_ptr(), L.color_rows.data_ptr(), cs, NCOLORS, r.data_ptr(),
                     x.data_ptr(), st)

    def _desc(self, lev: int):
        L = self.levels[lev]
        if L.desc is None:
            from .kernels import descriptor
            L.desc = descriptor(L.op)
        return L.desc

    def _spmv(self, lev: int, x, y, st=None) -> None:
        _native.call("ds_spmv", ctypes.byref(self._desc(lev)), x.data_ptr(), y.data_ptr(), 0,
                     self._stream() if st is None else st)

    def vcycle(self, r, z, lev: int = 0, st=None) -> None:
        """z = M^-1 r (ComputeMG_ref): z = 0; pre-smooth; restrict
        r - A z; recurse; prolong; post-smooth.  Coarsest: one smooth."""
        L = self.levels[lev]
        st = self._stream() if st is None else st
        z.zero_()                    # torch's current stream == st (eager or capture)
        self.symgs(lev, r, z, st)
        if L.f2c is None:
            return
        C = self.levels[lev + 1]
        nc = C.nrows
        if L.op.format_id == FormatId.DIA:
            # only the coarse rows of A z are formed (fused, bitwise equal)
            _native.call("ds_mg_restrict_residual", ctypes.byref(self._desc(lev)), nc,
                         L.f2c.data_ptr(), z.data_ptr(), r.data_ptr(), C.r.data_ptr(), st)
        else:
            self._spmv(lev, z, L.axf, st)
            _native.call("ds_mg_restrict", nc, L.f2c.data_ptr(), r.data_ptr(),
                         L.axf.data_ptr(), C.r.data_ptr(), st)
        self.vcycle(C.r, C.x, lev + 1, st)
        _native.call("ds_mg_prolong", nc, L.f2c.data_ptr(), C.x.data_ptr(), z.data_ptr(), st)
        self.symgs(lev, r, z, st)


_ELL_WIDTHS = (8, 16, 26, 32)
_OELL_MIN_ROWS = 1 << 20


def _ell(L: MgLevel, dev):
    """Colour-ordered ELL copy of the level operator (None if a row has more
    than 32 off-diagonals: the sweep then reads the CSR operator)."""
    import torch
    from . import _device
    a = L.a
    n = a.nrows
    st = _device.stream(dev)
    w = ctypes.c_int32()
    _native.call("ds_symgs_ell_width", n, a.row_offsets.data_ptr(), a.col_indices.data_ptr(),
                 ctypes.byref(w), st)
    width = next((v for v in _ELL_WIDTHS if v >= w.value), None)
    if width is None:
        return None
    ec = torch.empty(width * n, dtype=torch.int32, device=dev)
    ev = torch.empty(width * n, dtype=torch.float64, device=dev)
    el = torch.empty(n, dtype=torch.int32, device=dev)
    dg = torch.empty(n, dtype=torch.float64, device=dev)
    _native.call("ds_symgs_ell_fill", n, width, a.row_offsets.data_ptr(),
                 a.col_indices.data_ptr(), a.values.data_ptr(), L.color_rows.data_ptr(),
                 ec.data_ptr(), ev.data_ptr(), el.data_ptr(), dg.data_ptr(), st)
    return (width, ec, ev, el, dg)


def _oell(L: MgLevel, dev):
    """Offset-ELL copy of the level operator (ds_symgs_oell_fill): None when
    its off-diagonals fall on more than 32 distinct offsets."""
    import torch
    from . import _device
    a = L.a
    n = a.nrows
    ro = a.row_offsets.to(torch.int64)
    rows = torch.repeat_interleave(torch.arange(n, device=dev), ro[1:] - ro[:-1])
    d = a.col_indices.to(torch.int64) - rows
    u = torch.unique(d[d != 0])   # ascending
    del rows, d
    if u.numel() > 32:
        return None
    width = 26 if u.numel() <= 26 else 32
    offs = torch.zeros(width, dtype=torch.int32, device=dev)   # padding 0: never an off-diagonal
    offs[:u.numel()] = u.to(torch.int32)
    ov = torch.empty(width * n, dtype=torch.float64, device=dev)
    mk = torch.empty(n, dtype=torch.int32, device=dev)
    dg = torch.empty(n, dtype=torch.float64, device=dev)
    rc = _native.load().ds_symgs_oell_fill(
        n, width, offs.data_ptr(), a.row_offsets.data_ptr(), a.col_indices.data_ptr(),
        a.values.data_ptr(), L.color_rows.data_ptr(), ov.data_ptr(), mk.data_ptr(),
        dg.data_ptr(), _device.stream(dev))
    if rc == _native.DS_ERR_NOT_SUPPORTED:
        return None
    _native.check(rc)
    return (width, offs.cpu().numpy().copy(), ov, mk, dg)


def _t(v):
    return v.data if isinstance(v, DenseVector) else v


def symgs(h: MgHierarchy, r, x, level: int = 0) -> None:
    """Public SymGS on a hierarchy level; r, x are device DenseVectors or tensors."""
    rt, xt = _t(r), _t(x)
    n = h.levels[level].nrows
    if rt.numel() != n or xt.numel() != n:
        raise DimensionMismatch(f"vectors must have {n} entries")
    with _cuda(h.device):
        h.symgs(level, rt, xt)


def mg(h: MgHierarchy, r, z) -> None:
    """z = V-cycle(r) on the finest level."""
    rt, zt = _t(r), _t(z)
    n = h.levels[0].nrows
    if rt.numel() != n or zt.numel() != n:
        raise DimensionMismatch(f"vectors must have {n} entries")
    with _cuda(h.device):
        h.vcycle(rt, zt)


def _cuda(dev):
    import torch
    return torch.cuda.device(dev)


class PcgEngine:
    """HPCG's preconditioned CG (ComputeCG_ref) with every scalar on the
    device (ds_pcg_scalars), so an iteration -- SpMV, three dots, the
    V-cycle's ~120 launches and the guarded vector updates -- is one CUDA
    graph replay with no host round trip; the host reads the 80-byte scalar
    block once per chunk of iterations."""

    def __init__(self, h: MgHierarchy, b, x0=None, tol: float = 1e-9, max_iters: int = 50):
        import torch
        from . import _device
        self.h, self.dev = h, h.device
        n = self.n = h.levels[0].nrows
        bt = _t(b)
        if bt.numel() != n:
            raise DimensionMismatch(f"b has {bt.numel()} entries, operator {n}")
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.b = bt
        self.x = torch.zeros(n, **f64) if x0 is None else _t(x0).clone()
        self.r, self.z, self.p, self.ap = (torch.empty(n, **f64) for _ in range(4))
        self.tol, self.max_iters = float(tol), int(max_iters)
        self.hist = torch.zeros(self.max_iters + 1, **f64)
        self.scal = torch.zeros(ctypes.sizeof(_native.DsPcgScalars), dtype=torch.uint8,
                                device=self.dev)
        self.ws = _device.workspace(self.dev)
        self.graph = None

    def _sp(self, field: str) -> int:
        return self.scal.data_ptr() + getattr(_native.DsPcgScalars, field).offset

    def _dot(self, u, v, field: str, st) -> None:
        _native.call("ds_dot", self.n, u.data_ptr(), v.data_ptr(), self._sp(field),
                     self.ws.data_ptr(), st)

    def _axpy(self, w, x, coef: str, negate: int, y, st) -> None:
        _native.call("ds_pcg_axpy", self.n, w.data_ptr(), x.data_ptr(), self._sp(coef), negate,
                     y.data_ptr(), self.scal.data_ptr(), st)

    def scalars(self) -> _native.DsPcgScalars:
        return _native.DsPcgScalars.from_buffer_copy(self.scal.cpu().numpy().tobytes())

    def setup(self) -> bool:
        """r = b - A x0, ||b||, history[0], z = M r, p = z, r.z.  True if
        already converged (no iteration needed)."""
        import torch
        from . import _device
        h, n, st = self.h, self.n, _device.stream(self.dev)
        h._spmv(0, self.x, self.ap)
        _native.call("ds_waxpby", n, 1.0, self.b.data_ptr(), -1.0, self.ap.data_ptr(),
                     self.r.data_ptr(), st)
        self._dot(self.b, self.b, "rtz_new", st)          # scratch slots for bb, rr
        self._dot(self.r, self.r, "rr", st)
        sc = self.scalars()
        bb, rr = sc.rtz_new, sc.rr
        nb = math.sqrt(bb)
        scale = nb if nb > 0.0 else 1.0
        h0 = math.sqrt(rr) / scale
        init = _native.DsPcgScalars(rr=rr, scale=scale, tol=self.tol,
                                    max_iters=self.max_iters, done=1 if h0 <= self.tol else 0)
        self.scal.copy_(torch.frombuffer(bytearray(bytes(init)), dtype=torch.uint8))
        self.hist[0] = h0
        if init.done:
            return True
        h.vcycle(self.r, self.z)
        _native.call("ds_waxpby", n, 1.0, self.z.data_ptr(), 0.0, self.z.data_ptr(),
                     self.p.data_ptr(), st)
        self._dot(self.r, self.z, "rtz", st)
        return False

    def step(self, st) -> None:
        h = self.h
        h._spmv(0, self.p, self.ap, st)
        self._dot(self.p, self.ap, "pap", st)
        _native.call("ds_pcg_alpha", self.scal.data_ptr(), st)
        self._axpy(self.x, self.x, "alpha", 0, self.p, st)
        self._axpy(self.r, self.r, "alpha", 1, self.ap, st)
        self._dot(self.r, self.r, "rr", st)
        _native.call("ds_pcg_check", self.scal.data_ptr(), self.hist.data_ptr(), st)
        h.vcycle(self.r, self.z, 0, st)
        self._dot(self.r, self.z, "rtz_new", st)
        _native.call("ds_pcg_beta", self.scal.data_ptr(), st)
        self._axpy(self.p, self.z, "beta", 0, self.p, st)

    def _capture(self, c: int) -> None:
        import torch
        from . import _device
        cap = torch.cuda.Stream(self.dev)
        cap.wait_stream(torch.cuda.current_stream(self.dev))
        ws = _device.new_workspace(self.dev)   # owned by this graph (kept on the engine)
        torch.cuda.synchronize(self.dev)
        saved, self.ws = self.ws, ws
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            for _ in range(c):
                self.step(cap.cuda_stream)
        self.ws = saved
        self.graph = g
        self._graph_ws = ws

    def run(self, use_graph: bool = True, chunk: int = 4) -> CgResult:
        from . import _device
        with _cuda(self.dev):
            if not self.setup():
                if use_graph and self.graph is None:
                    self._capture(chunk)
                rounds = 1
                while True:
                    for _ in range(rounds):
                        if use_graph:
                            self.graph.replay()
                        else:
                            st = _device.stream(self.dev)
                            for _ in range(chunk):
                                self.step(st)
                    sc = self.scalars()
                    if sc.done:
                        break
                    rounds = min(rounds * 2, 8)
            sc = self.scalars()
            if sc.done == 2:
                raise BreakdownZeroCurvature(f"p'Ap = {sc.pap} at iteration {sc.iter + 1}")
            hist = self.hist[:sc.iter + 1].cpu().numpy().copy()
        return CgResult(DenseVector(self.x), int(sc.iter), hist, sc.done == 1)


def pcg(h: MgHierarchy, b, x0=None, tol: float = 1e-9, max_iters: int = 50,
        use_graph: bool = True) -> CgResult:
    """HPCG's preconditioned CG (ComputeCG_ref) with the MG preconditioner.
    History = ||r|| / ||b|| per iteration, like ``cg`` (solver.py:56-189)."""
    return PcgEngine(h, b, x0, tol, max_iters).run(use_graph=use_graph)
