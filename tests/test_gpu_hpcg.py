"""GPU parity of the HPCG smoother / multigrid / PCG
against the oracle's restatement (oracle.symgs_colored, mg_vcycle, pcg_mg).

The reference has no SymGS/MG, so parity here is pinned to the
oracle only.  Bar: SymGS sweeps and V-cycles BITWISE equal; PCG iterations
equal and residual history within 1e-8 relative (dots are a fixed tree on
the device, np.dot on the host -- the tolerance of the CG tests).
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_2209_06478_b200 import hpcg  # noqa: E402
from oracle import dynsparse_oracle as O  # noqa: E402

DEV = torch.device("cuda", 0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(DEV)


@pytest.mark.parametrize("layout", ["oell", "ell-cols", "ell", "csr"])
@pytest.mark.parametrize("dims", [(8, 8, 8), (5, 6, 7), (16, 8, 4), (1, 1, 3), (2, 1, 1)])
def test_symgs_bitwise(dims, layout):
    nx, ny, nz = dims
    h = hpcg.MgHierarchy.build(nx, ny, nz, nlevels=1, device=DEV, layout=layout)
    # "oell": the offset ELL (the stencil's off-diagonals fall on <= 26
    # offsets); "ell" picks it only from 2^20 rows, the column ELL below
    assert (h.levels[0].oell is not None) == (layout == "oell")
    assert (h.levels[0].ell is not None) == (layout in ("ell-cols", "ell"))
    m = O.stencil_partition(nx, ny, nz).a_full
    rng = np.random.default_rng(sum(dims))
    r = rng.standard_normal(m.nrows)
    x = rng.standard_normal(m.nrows)
    xd = dev(x)
    for _ in range(2):
        O.symgs_colored(m, r, x, O.stencil_colors(nx, ny, nz))
        hpcg.symgs(h, dev(r), xd)
        assert xd.cpu().numpy().tobytes() == x.tobytes()


@pytest.mark.parametrize("dims", [(16, 16, 16), (8, 12, 16)])
@pytest.mark.parametrize("layout,fmt", [("ell", "dia"), ("csr", "csr"), ("ell", "coo"),
                                        ("oell", "dia")])
def test_vcycle_bitwise(dims, layout, fmt):
    h = hpcg.MgHierarchy.build(*dims, nlevels=4, device=DEV, layout=layout, spmv_format=fmt)
    levels = O.mg_levels(*dims, levels=4, fmt={"dia": O.DIA, "csr": O.CSR, "coo": O.COO}[fmt])
    assert [L.nrows for L in h.levels] == [lv[0].nrows for lv in levels]
    rng = np.random.default_rng(7)
    r = rng.standard_normal(levels[0][0].nrows)
    z = np.zeros_like(r)
    O.mg_vcycle(levels, 0, r, z)
    zd = torch.full_like(dev(r), 123.0)         # the V-cycle zeroes z itself
    hpcg.mg(h, dev(r), zd)
    assert zd.cpu().numpy().tobytes() == z.tobytes()


def test_symgs_large_level_layouts_agree():
    """A level spanning many CTAs per colour: ELL and CSR sweeps and the
    restatement agree bit for bit over repeated sweeps."""
    dims = (48, 40, 36)
    m = O.stencil_partition(*dims).a_full
    rng = np.random.default_rng(5)
    r, x = rng.standard_normal(m.nrows), rng.standard_normal(m.nrows)
    outs = []
    for layout in ("oell", "ell-cols", "csr"):
        h = hpcg.MgHierarchy.build(*dims, nlevels=1, device=DEV, layout=layout)
        xd = dev(x)
        for _ in range(3):
            hpcg.symgs(h, dev(r), xd)
        outs.append(xd.cpu().numpy())
    assert outs[0].tobytes() == outs[1].tobytes() == outs[2].tobytes()
    ref = x.copy()
    O.symgs_colored(m, r, ref, O.stencil_colors(*dims))
    h = hpcg.MgHierarchy.build(*dims, nlevels=1, device=DEV)
    xd = dev(x)
    hpcg.symgs(h, dev(r), xd)
    assert xd.cpu().numpy().tobytes() == ref.tobytes()


@pytest.mark.parametrize("layout", ["oell", "ell-cols"])
def test_symgs_signed_zero_and_padding(layout):
    """Padding / absent slots never touch the arithmetic: r = -0 rows with
    x = -0 neighbours keep their signed zeros exactly like the CSR walk (the
    offset ELL's absent slots hold 0.0 and gather real x values: both are
    selected away by the presence mask)."""
    dims = (3, 3, 3)                      # corner rows have 7 entries, pad to 26
    h = hpcg.MgHierarchy.build(*dims, nlevels=1, device=DEV, layout=layout)
    L = h.levels[0]
    assert (L.oell if layout == "oell" else L.ell)[0] == 26
    m = O.stencil_partition(*dims).a_full
    r = np.full(m.nrows, -0.0)
    x = np.full(m.nrows, -0.0)
    x[::5] = -1.0
    xd = dev(x)
    O.symgs_colored(m, r, x, O.stencil_colors(*dims))
    hpcg.symgs(h, dev(r), xd)
    assert xd.cpu().numpy().tobytes() == x.tobytes()


@pytest.mark.parametrize("use_graph", [True, False])
def test_pcg_matches_oracle_and_beats_cg(use_graph):
    dims = (16, 16, 16)
    h = hpcg.MgHierarchy.build(*dims, device=DEV)
    levels = O.mg_levels(*dims, fmt=O.DIA)
    b = O.stencil_partition(*dims).b
    ref = O.pcg_mg(levels, b, tol=1e-9, max_iters=50)
    res = hpcg.pcg(h, dev(b), tol=1e-9, max_iters=50, use_graph=use_graph)
    assert res.converged and ref.converged
    assert res.iterations == ref.iterations
    rel = np.abs(res.residual_history - ref.history) / np.abs(ref.history)
    assert rel.max() < 1e-8, rel.max()
    x = res.x.data.cpu().numpy()
    assert np.abs(x - 1.0).max() < 1e-7          # xexact = ones
    plain = O.cg(O.stencil_partition(*dims).a_full, b, tol=1e-9)
    assert res.iterations < plain.iterations


def test_pcg_max_iters_and_zero_rhs():
    dims = (8, 8, 8)
    h = hpcg.MgHierarchy.build(*dims, device=DEV)
    levels = O.mg_levels(*dims, fmt=O.DIA)
    b = O.stencil_partition(*dims).b
    ref = O.pcg_mg(levels, b, tol=1e-30, max_iters=3)
    res = hpcg.pcg(h, dev(b), tol=1e-30, max_iters=3)      # graph chunk of 4 overshoots
    assert res.iterations == 3 and not res.converged and res.residual_history.size == 4
    assert np.allclose(res.residual_history, ref.history, rtol=1e-8, atol=0)
    z = hpcg.pcg(h, dev(np.zeros_like(b)))
    assert z.converged and z.iterations == 0 and not z.x.data.abs().sum().item()


def test_symgs_offset_ell_at_hpcg_size():
    """104^3 (the bench's level 0, >= 2^20 rows): the default layout takes the
    offset ELL and its sweep is bitwise the column ELL's and the restatement's."""
    dims = (104, 104, 104)
    h = hpcg.MgHierarchy.build(*dims, nlevels=1, device=DEV)
    assert h.levels[0].oell is not None and h.levels[0].ell is None
    hc = hpcg.MgHierarchy.build(*dims, nlevels=1, device=DEV, layout="ell-cols")
    rng = np.random.default_rng(104)
    n = h.levels[0].nrows
    r, x = rng.standard_normal(n), rng.standard_normal(n)
    xa, xb = dev(x), dev(x)
    for _ in range(2):
        hpcg.symgs(h, dev(r), xa)
        hpcg.symgs(hc, dev(r), xb)
    assert xa.cpu().numpy().tobytes() == xb.cpu().numpy().tobytes()
    m = O.stencil_partition(*dims).a_full
    ref = x.copy()
    cols = O.stencil_colors(*dims)
    for _ in range(2):
        O.symgs_colored(m, r, ref, cols)
    assert xa.cpu().numpy().tobytes() == ref.tobytes()
