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


@pytest.mark.parametrize("dims", [(8, 8, 8), (5, 6, 7), (16, 8, 4), (1, 1, 3)])
def test_symgs_bitwise(dims):
    nx, ny, nz = dims
    h = hpcg.MgHierarchy.build(nx, ny, nz, nlevels=1, device=DEV)
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
def test_vcycle_bitwise(dims):
    h = hpcg.MgHierarchy.build(*dims, nlevels=4, device=DEV)
    levels = O.mg_levels(*dims, levels=4)
    assert [L.nrows for L in h.levels] == [lv[0].nrows for lv in levels]
    rng = np.random.default_rng(7)
    r = rng.standard_normal(levels[0][0].nrows)
    z = np.zeros_like(r)
    O.mg_vcycle(levels, 0, r, z)
    zd = torch.full_like(dev(r), 123.0)         # the V-cycle zeroes z itself
    hpcg.mg(h, dev(r), zd)
    assert zd.cpu().numpy().tobytes() == z.tobytes()


def test_pcg_matches_oracle_and_beats_cg():
    dims = (16, 16, 16)
    h = hpcg.MgHierarchy.build(*dims, device=DEV)
    levels = O.mg_levels(*dims)
    b = O.stencil_partition(*dims).b
    ref = O.pcg_mg(levels, b, tol=1e-9, max_iters=50)
    res = hpcg.pcg(h, dev(b), tol=1e-9, max_iters=50)
    assert res.converged and ref.converged
    assert res.iterations == ref.iterations
    rel = np.abs(res.residual_history - ref.history) / np.abs(ref.history)
    assert rel.max() < 1e-8, rel.max()
    x = res.x.data.cpu().numpy()
    assert np.abs(x - 1.0).max() < 1e-7          # xexact = ones
    plain = O.cg(O.stencil_partition(*dims).a_full, b, tol=1e-9)
    assert res.iterations < plain.iterations
