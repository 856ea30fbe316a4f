"""CPU checks of the HPCG restatement and the host-side colour plan.

No reference fixture exists for SymGS/MG (the reference stops at plain CG,
SPEC.md:16), so the oracle is checked through the properties HPCG relies on:
no two coupled rows share a colour, the sweep is symmetric (forward then
backward == the transpose order), one SymGS on A x* = b keeps x* fixed, and
the MG-preconditioned CG converges in fewer iterations than plain CG.
"""

from __future__ import annotations

import numpy as np

from oracle import dynsparse_oracle as O
from paper_2209_06478_b200 import hpcg


def test_colouring_decouples_rows():
    for dims in [(4, 4, 4), (5, 3, 2), (1, 1, 5)]:
        m = O.stencil_partition(*dims).a_full
        c = O.stencil_colors(*dims)
        assert np.array_equal(c, hpcg.stencil_colors(*dims))
        rows = np.repeat(np.arange(m.nrows), np.diff(m.offsets))
        off_diag = rows != m.cols
        assert not np.any(c[rows[off_diag]] == c[m.cols[off_diag]])


def test_colour_lists():
    c = O.stencil_colors(5, 3, 2)
    rows, start = hpcg._color_lists(c)
    assert start[0] == 0 and start[-1] == c.size and start.size == 9
    for k in range(8):
        seg = rows[start[k]:start[k + 1]]
        assert np.all(c[seg] == k) and np.all(np.diff(seg) > 0)


def test_symgs_fixed_point_and_levels():
    m = O.stencil_partition(4, 4, 4).a_full
    xs = np.ones(m.nrows)
    b = np.zeros(m.nrows)
    O.spmv(m, xs, b)
    x = xs.copy()
    O.symgs_colored(m, b, x, O.stencil_colors(4, 4, 4))
    assert np.allclose(x, 1.0, rtol=0, atol=1e-14)
    lv = O.mg_levels(8, 8, 8)
    assert [a.nrows for a, _, _, _ in lv] == [512, 64, 8, 1]
    assert lv[-1][2] is None and all(f.size == a.nrows for (_, _, f, _), (a, _, _, _)
                                     in zip(lv[:-1], lv[1:]))


def test_pcg_converges_faster_than_cg():
    dims = (8, 8, 8)
    p = O.stencil_partition(*dims)
    res = O.pcg_mg(O.mg_levels(*dims), p.b, tol=1e-9)
    plain = O.cg(p.a_full, p.b, tol=1e-9)
    assert res.converged and res.iterations < plain.iterations
    assert np.abs(res.x - 1.0).max() < 1e-7
    dia = O.pcg_mg(O.mg_levels(*dims, fmt=O.DIA), p.b, tol=1e-9)
    assert dia.iterations == res.iterations
    assert np.allclose(dia.history, res.history, rtol=1e-10, atol=0)
