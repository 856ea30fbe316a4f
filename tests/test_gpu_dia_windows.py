"""DIA SpMV with the TMA-staged x windows (ds_dia.cu dia_issue_windows),
forced at small sizes in a subprocess (the launcher reads DS_DIA_XWIN_FORCE /
DS_DIA_XWIN_SPAN once): bitwise equal to the oracle on stencils whose edges
clip the windows (odd and even column counts, ragged last tiles), spmv_add,
and inside CG (the windows are issued after the programmatic-launch wait);
unsorted offsets fall back to plain gathers."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r'''
import numpy as np, torch
import paper_2209_06478_b200 as ds
from oracle import dynsparse_oracle as O
dev = torch.device("cuda", 0)
for dims in [(24, 20, 16), (9, 7, 5), (33, 17, 11), (40, 40, 40)]:
    part = ds.generate_problem(ds.GridSpec(*dims)).partitions[0]
    A = ds.convert(ds.to_device(part.a_full, dev), ds.FormatId.DIA)
    ref = O.convert(O.stencil_partition(*dims).a_full, O.DIA)
    rng = np.random.default_rng(sum(dims))
    x = rng.standard_normal(A.ncols)
    for acc in (False, True):
        y0 = rng.standard_normal(A.nrows)
        y = ds.DenseVector(torch.from_numpy(y0.copy()).to(dev))
        (ds.spmv_add if acc else ds.spmv)(ds.SERIAL, A, ds.DenseVector(torch.from_numpy(x).to(dev)), y)
        want = y0.copy()
        (O.spmv_add if acc else O.spmv)(ref, x, want)
        assert y.data.cpu().numpy().tobytes() == want.tobytes(), (dims, acc)
    res = ds.cg(ds.SERIAL, A, ds.to_device(part.b, dev), tol=1e-9, max_iters=500)
    oref = O.cg(ref, O.stencil_partition(*dims).b, tol=1e-9, max_iters=500)
    assert res.converged and abs(res.iterations - oref.iterations) <= 1, dims
    k = min(res.iterations, oref.iterations) + 1
    h = np.asarray(res.residual_history[:k])
    assert np.all(np.abs(h - oref.history[:k]) <= 1e-8 * oref.history[:k] + 1e-14), dims
# unsorted offsets (the same 27 diagonals permuted): no windows, j-order sums
rng = np.random.default_rng(5)
perm = rng.permutation(27)
offs = A.offsets.cpu().numpy()[perm]
vals = np.ascontiguousarray(A.values.cpu().numpy()[:, perm])
Ap = ds.DiaMatrix(A.nrows, A.ncols, offs, vals, ds.MemorySpace.DEVICE, dev)
refp = O.dia(A.nrows, A.ncols, offs, vals)
x = rng.standard_normal(A.ncols)
y = ds.DenseVector.zeros(A.nrows, ds.MemorySpace.DEVICE, dev)
ds.spmv(ds.SERIAL, Ap, ds.DenseVector(torch.from_numpy(x).to(dev)), y)
want = np.zeros(A.nrows)
O.spmv(refp, x, want)
assert y.data.cpu().numpy().tobytes() == want.tobytes(), "permuted offsets"
print("ok")
'''


def test_dia_windows_forced_bitwise():
    env = dict(os.environ, DS_DIA_XWIN_FORCE="1", DS_DIA_XWIN_SPAN="0",
               PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
