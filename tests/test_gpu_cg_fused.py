"""The single-partition CG iteration with the fused update + direction kernel
(ds_cg_update_direction_deferred: grid barrier between the two phases)
against the two-kernel path and the reference (golden KATs): iterations,
residual history and x (solver.py:170-188; test_solver.py:78-83, 121)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import kat

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2209_06478_b200 as ds  # noqa: E402
from paper_2209_06478_b200 import _native  # noqa: E402
from oracle import dynsparse_oracle as O  # noqa: E402

DEV = torch.device("cuda", 0)


def _solve(a, b, monkeypatch, fused, **kw):
    if fused:
        monkeypatch.delenv("DS_CG_UNFUSED", raising=False)
    else:
        monkeypatch.setenv("DS_CG_UNFUSED", "1")
    return ds.cg(ds.SERIAL, ds.DynamicMatrix(a), b, **kw)


@pytest.mark.parametrize("fmt", ["csr", "dia", "coo"])
def test_fused_matches_reference_and_unfused(fmt, monkeypatch):
    K = kat()
    part = ds.generate_problem(ds.GridSpec(16, 16, 16), space=ds.MemorySpace.DEVICE,
                               device=DEV).partitions[0]
    a = ds.convert(part.a_full, ds.FormatId[fmt.upper()])
    fused = _solve(a, part.b, monkeypatch, True, tol=1e-9, max_iters=500)
    plain = _solve(a, part.b, monkeypatch, False, tol=1e-9, max_iters=500)
    it_ref = int(K[f"cg16/{fmt}/iters"][0])
    h_ref = K[f"cg16/{fmt}/hist"]
    for res in (fused, plain):
        assert res.converged and abs(res.iterations - it_ref) <= 1
        k = min(res.iterations, it_ref) + 1
        h = np.asarray(res.residual_history[:k])
        assert np.all(np.abs(h - h_ref[:k]) <= 1e-8 * h_ref[:k] + 64 * np.finfo(float).eps)
        x = res.x.data.cpu().numpy()
        assert np.max(np.abs(x - K[f"cg16/{fmt}/x"])) < 1e-8
    # the two device paths differ only in the r.r reduction tree
    assert fused.iterations == plain.iterations
    hf, hp = np.asarray(fused.residual_history), np.asarray(plain.residual_history)
    assert np.all(np.abs(hf - hp) <= 1e-12 * hp + 64 * np.finfo(float).eps)


def test_fused_max_iters_and_odd_n(monkeypatch):
    """max_iters stop (done = 3) and an odd vector length (scalar tail)."""
    spec = ds.GridSpec(9, 7, 5)   # n = 315, odd
    part = ds.generate_problem(spec, space=ds.MemorySpace.DEVICE, device=DEV).partitions[0]
    ref = O.stencil_partition(9, 7, 5)
    for max_iters in (3, 500):
        res = _solve(part.a_full, part.b, monkeypatch, True, tol=1e-12, max_iters=max_iters)
        oref = O.cg(ref.a_full, ref.b, tol=1e-12, max_iters=max_iters)
        assert abs(res.iterations - oref.iterations) <= 1
        assert res.converged == oref.converged
        k = min(res.iterations, oref.iterations) + 1
        h = np.asarray(res.residual_history[:k])
        assert np.all(np.abs(h - oref.history[:k]) <= 1e-8 * oref.history[:k]
                      + 64 * np.finfo(float).eps)


def test_fused_entry_reports_unsupported_for_misaligned():
    lib = _native.load()
    n = 101
    buf = torch.zeros(4 * n + 1, dtype=torch.float64, device=DEV)
    x = buf.data_ptr() + 8   # 8-byte offset: not 16-byte aligned
    rc = lib.ds_cg_update_direction_deferred(n, x, x, x, x, None, None, None, None)
    assert rc == _native.DS_ERR_NOT_SUPPORTED


def test_l2_persist_window_fits_or_refuses():
    """ds_l2_persist takes whole windows only: a small one is set (and the
    reset gives the carve-out back); one larger than the persisting L2 is
    refused without side effects."""
    lib = _native.load()
    st = torch.cuda.current_stream(DEV).cuda_stream
    small = torch.zeros(1 << 20, dtype=torch.float64, device=DEV)          # 8 MB
    assert lib.ds_l2_persist(small.data_ptr(), small.numel() * 8, st) == 0
    assert lib.ds_l2_persist_reset(st) == 0
    huge_bytes = 1 << 40
    assert lib.ds_l2_persist(small.data_ptr(), huge_bytes, st) == _native.DS_ERR_NOT_SUPPORTED
    assert lib.ds_l2_persist_reset(st) == 0
