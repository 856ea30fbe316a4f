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
from .formats import CsrMatrix, DenseVector, MemorySpace
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

    @property
    def nrows(self) -> int:
        return self.a.nrows


@dataclass
class MgHierarchy:
    levels: list[MgLevel] = field(default_factory=list)
    device: object = None

    @staticmethod
    def build(nx: int, ny: int, nz: int, nlevels: int = 4, device=None) -> "MgHierarchy":
        """GenerateProblem + GenerateCoarseProblem: each coarse grid halves
        every dimension while all three stay even (at most ``nlevels``)."""
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
            if not coarsen:
                break
            nx, ny, nz = nx // 2, ny // 2, nz // 2
        return h

    # -- kernels ----------------------------------------------------------
    def _stream(self):
        from . import _device
        return _device.stream(self.device)

    def symgs(self, lev: int, r, x) -> None:
        """One symmetric colour sweep in place on level ``lev`` (ds_symgs)."""
        L = self.levels[lev]
        a = L.a
        st = L.color_start
        _native.call("ds_symgs", a.nrows, a.row_offsets.data_ptr(), a.col_indices.data_ptr(),
                     a.values.data_ptr(), L.color_rows.data_ptr(),
                     st.ctypes.data_as(_native.P_i64), NCOLORS, r.data_ptr(), x.data_ptr(),
                     self._stream())

    def _spmv(self, lev: int, x, y) -> None:
        from .kernels import descriptor
        d = descriptor(self.levels[lev].a)
        _native.call("ds_spmv", ctypes.byref(d), x.data_ptr(), y.data_ptr(), 0, self._stream())

    def vcycle(self, r, z, lev: int = 0) -> None:
        """z = M^-1 r (ComputeMG_ref): z = 0; pre-smooth; restrict
        r - A z; recurse; prolong; post-smooth.  Coarsest: one smooth."""
        L = self.levels[lev]
        z.zero_()
        self.symgs(lev, r, z)
        if L.f2c is None:
            return
        C = self.levels[lev + 1]
        st = self._stream()
        self._spmv(lev, z, L.axf)
        nc = C.nrows
        _native.call("ds_mg_restrict", nc, L.f2c.data_ptr(), r.data_ptr(), L.axf.data_ptr(),
                     C.r.data_ptr(), st)
        self.vcycle(C.r, C.x, lev + 1)
        _native.call("ds_mg_prolong", nc, L.f2c.data_ptr(), C.x.data_ptr(), z.data_ptr(), st)
        self.symgs(lev, r, z)


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


def pcg(h: MgHierarchy, b, x0=None, tol: float = 1e-9, max_iters: int = 50) -> CgResult:
    """HPCG's preconditioned CG (ComputeCG_ref) with the MG preconditioner.
    History = ||r|| / ||b|| per iteration, like ``cg`` (solver.py:56-189)."""
    import torch
    from . import _device
    dev = h.device
    n = h.levels[0].nrows
    bt = _t(b)
    if bt.numel() != n:
        raise DimensionMismatch(f"b has {bt.numel()} entries, operator {n}")
    with _cuda(dev):
        st = _device.stream(dev)
        ws = _device.workspace(dev)
        f64 = dict(dtype=torch.float64, device=dev)
        x = torch.zeros(n, **f64) if x0 is None else _t(x0).clone()
        r, z, p, ap = (torch.empty(n, **f64) for _ in range(4))
        dots = torch.zeros(3, **f64)

        def ddot(u, v, k):
            _native.call("ds_dot", n, u.data_ptr(), v.data_ptr(), dots[k:].data_ptr(),
                         ws.data_ptr(), st)

        def wax(al, u, be, v, w):
            _native.call("ds_waxpby", n, float(al), u.data_ptr(), float(be), v.data_ptr(),
                         w.data_ptr(), st)

        h._spmv(0, x, ap)
        wax(1.0, bt, -1.0, ap, r)
        ddot(bt, bt, 0)
        ddot(r, r, 1)
        bb, rr = dots[:2].tolist()
        nb = math.sqrt(bb)
        scale = nb if nb > 0.0 else 1.0
        hist = [math.sqrt(rr) / scale]
        if hist[0] <= tol:
            return CgResult(DenseVector(x), 0, np.asarray(hist), True)
        h.vcycle(r, z)
        wax(1.0, z, 0.0, z, p)
        ddot(r, z, 2)
        rtz = float(dots[2].item())
        it, done = 0, False
        for k in range(1, max_iters + 1):
            it = k
            h._spmv(0, p, ap)
            ddot(p, ap, 0)
            pap = float(dots[0].item())
            if pap <= 0.0:
                raise BreakdownZeroCurvature(f"p'Ap = {pap} at iteration {k}")
            alpha = rtz / pap
            wax(1.0, x, alpha, p, x)
            wax(1.0, r, -alpha, ap, r)
            ddot(r, r, 1)
            hist.append(math.sqrt(float(dots[1].item())) / scale)
            if hist[-1] <= tol:
                done = True
                break
            h.vcycle(r, z)
            ddot(r, z, 2)
            rtz_new = float(dots[2].item())
            wax(1.0, z, rtz_new / rtz, p, p)
            rtz = rtz_new
        return CgResult(DenseVector(x), it, np.asarray(hist), done)
