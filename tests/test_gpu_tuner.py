"""GPU: the per-partition format tuner (tuner.py:53-180) on device matrices --
every combination converted in place, CUDA-event timing, CSR restored,
remote DIA overflow skipped, selection rules as in the reference."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2209_06478_b200 as ds  # noqa: E402

F = ds.FormatId


def test_profile_and_select_on_device():
    dev = torch.device("cuda", 0)
    spec = ds.GridSpec(12, 12, 12, 2, 1, 1)
    prob = ds.generate_problem(spec, space=ds.MemorySpace.DEVICE, device=dev)
    splits = [ds.split_local_remote(prob, k) for k in range(prob.npartitions)]
    table = ds.profile_formats(ds.SERIAL, prob, splits, reps=3)
    assert table.npartitions == 2
    for k in range(2):
        for lf in F:
            for rf in F:
                cell = (k, lf, rf)
                assert (cell in table.entries) != (cell in table.skipped)
                if cell in table.entries:
                    assert table.entries[cell] > 0
        assert (k, F.CSR, F.DIA) in table.skipped      # the remote part overflows DIA
    for sp in splits:                                  # restored to CSR
        assert sp.local.active is F.CSR and sp.remote.active is F.CSR
    multi = ds.select_plan(table, "multi")
    for k, (lf, rf) in enumerate(multi.assignments):
        best = min(v for (kk, _, _), v in table.entries.items() if kk == k)
        assert table.entries[(k, lf, rf)] == best
    assert ds.select_plan(table, "fixed").assignments == [(F.CSR, F.CSR)] * 2
    # the plan is applied and the distributed solve still matches the reference rules
    for sp, (lf, rf) in zip(splits, multi.assignments):
        ds.convert_inplace(sp.local, lf)
        ds.convert_inplace(sp.remote, rf)
    res = ds.cg(ds.SERIAL, ds.DistributedOperator(prob, splits), [p.b for p in prob.partitions])
    assert res.converged
