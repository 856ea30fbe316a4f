"""CPU: the tuner's selection rules and CSV contract (reference
tuner.py:123-224, tests test_tuner.py:38-140) on synthetic timing tables,
checked against the oracle's restatement and -- when /root/reference is
mounted -- the reference's own select_plan; plus the amortised
conversion-cost selection (new)."""

from __future__ import annotations

import itertools
import os
import sys

import numpy as np
import pytest

import paper_2209_06478_b200 as ds
from paper_2209_06478_b200 import tuner as T
from oracle import dynsparse_oracle as O

F = ds.FormatId
REF = "/root/reference/pkg/src"


def _random_table(rng, nparts, p_skip=0.2, ties=False):
    t = T.TimingTable(entries={}, reps=5, npartitions=nparts)
    for k, lf, rf in itertools.product(range(nparts), T.FORMATS, T.FORMATS):
        if rng.random() < p_skip:
            t.skipped.add((k, lf, rf))
        else:
            v = float(rng.integers(1, 4)) if ties else float(rng.random())
            t.entries[(k, lf, rf)] = v * 1e-4
    return t


def _oracle_plan(t, mode):
    e = {(k, int(lf), int(rf)): v for (k, lf, rf), v in t.entries.items()}
    return [(F(a), F(b)) for a, b in O.select_plan(e, t.npartitions, mode)]


@pytest.mark.parametrize("ties", [False, True])
def test_select_plan_matches_oracle(ties):
    rng = np.random.default_rng(7 + ties)
    for _ in range(200):
        t = _random_table(rng, int(rng.integers(1, 6)), ties=ties)
        for mode in ("multi", "morpheus", "ghost"):
            try:
                want = _oracle_plan(t, mode)
            except ValueError:
                with pytest.raises(ds.EmptySearchSpace):
                    T.select_plan(t, mode)
                continue
            assert T.select_plan(t, mode).assignments == want, (mode, t.entries)


def test_fixed_needs_csr_everywhere_and_unknown_mode():
    t = T.TimingTable(entries={(0, F.CSR, F.CSR): 1.0, (1, F.DIA, F.CSR): 1.0}, reps=1,
                      npartitions=2)
    with pytest.raises(ds.EmptySearchSpace):
        T.select_plan(t, "fixed")
    t.entries[(1, F.CSR, F.CSR)] = 2.0
    assert T.select_plan(t, "fixed").assignments == [(F.CSR, F.CSR)] * 2
    with pytest.raises(ValueError):
        T.select_plan(t, "fastest")


def test_amortised_switch_cost_changes_the_pick():
    """DIA is 10% faster per SpMV but costs 5 SpMVs to switch to: worth it
    for a long solve, not for a short one; without iterations the pick is
    the reference's (SpMV time only)."""
    t = T.TimingTable(entries={(0, F.CSR, F.CSR): 1.0e-4, (0, F.DIA, F.CSR): 0.9e-4},
                      reps=1, npartitions=1,
                      convert_seconds={(0, F.CSR, F.CSR): 0.0, (0, F.DIA, F.CSR): 5.0e-4})
    assert T.select_plan(t, "multi").assignments == [(F.DIA, F.CSR)]
    assert T.select_plan(t, "multi", iterations=1000).assignments == [(F.DIA, F.CSR)]
    assert T.select_plan(t, "multi", iterations=10).assignments == [(F.CSR, F.CSR)]
    assert T.select_plan(t, "morpheus", iterations=10).assignments == [(F.CSR, F.CSR)]


def test_csv_roundtrip(tmp_path):
    rng = np.random.default_rng(3)
    t = _random_table(rng, 3)
    path = tmp_path / "table.csv"
    T.write_timing_table(t, path)
    back = T.read_timing_table(path)
    assert back.npartitions == 3 and back.reps == 5
    assert back.skipped == t.skipped
    assert set(back.entries) == set(t.entries)
    for cell, v in t.entries.items():
        assert back.entries[cell] == pytest.approx(v, rel=1e-9)
    header = path.read_text().splitlines()[0]
    assert header == ",".join(T.TIMING_TABLE_COLUMNS)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_select_plan_and_csv_match_live_reference(tmp_path):
    sys.path.insert(0, REF)
    try:
        import dynsparse as R
        from dynsparse import tuner as RT
    finally:
        sys.path.remove(REF)
    rng = np.random.default_rng(11)
    for _ in range(100):
        t = _random_table(rng, int(rng.integers(1, 5)), ties=bool(rng.integers(0, 2)))
        rt = RT.TimingTable(
            entries={(k, R.FormatId(int(a)), R.FormatId(int(b))): v
                     for (k, a, b), v in t.entries.items()},
            reps=t.reps, skipped={(k, R.FormatId(int(a)), R.FormatId(int(b)))
                                  for (k, a, b) in t.skipped}, npartitions=t.npartitions)
        for mode in ("multi", "morpheus", "ghost", "fixed"):
            try:
                want = [(int(a), int(b)) for a, b in RT.select_plan(rt, mode).assignments]
            except R.EmptySearchSpace:
                with pytest.raises(ds.EmptySearchSpace):
                    T.select_plan(t, mode)
                continue
            got = [(int(a), int(b)) for a, b in T.select_plan(t, mode).assignments]
            assert got == want, mode
    # the CSV files are byte-identical
    RT.write_timing_table(rt, tmp_path / "ref.csv")
    T.write_timing_table(t, tmp_path / "ours.csv")
    assert (tmp_path / "ref.csv").read_bytes() == (tmp_path / "ours.csv").read_bytes()
