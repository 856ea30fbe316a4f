"""dynsparse-bench (paper_2209_06478_b200.runbench) against the reference's
harness contract (reference tests/test_bench.py): phase order, partial
reports, validation gating, JSON / CSV emission, CLI flags and exit codes.
CPU tests: argument errors and report emission; GPU tests: the phases."""

from __future__ import annotations

import csv
import json
import os
import subprocess
import sys

import pytest

import paper_2209_06478_b200 as ds
from paper_2209_06478_b200 import runbench as RB
from paper_2209_06478_b200.solver import ValidationReport

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2209_06478_b200.runbench", *args],
                          capture_output=True, text=True, timeout=600, cwd=ROOT)


def _synthetic_report(error=False):
    rep = RB.RunReport(config=RB.BenchConfig(nx=4, ny=4, nz=4, procs=(2, 1, 1)).echo(),
                       setup_seconds=0.5, reference_spmv_seconds=0.25)
    rep.partitions = [{"partition": k, "local_format": "csr", "remote_format": "csr",
                       "local_nnz": 10, "remote_nnz": 3, "remote_empty": False}
                      for k in range(2)]
    if error:
        rep.error = {"phase": "optimization_setup", "partition": 0, "local_format": "csr",
                     "remote_format": "dia", "message": "DiaFillOverflow"}
    else:
        rep.validation = {"passed": True, "converged": True, "iterations": 3,
                          "iteration_bound": 12, "final_residual": 1e-13}
        rep.optimized_spmv_seconds, rep.spmv_ratio = 0.125, 2.0
    return rep


def test_cli_argument_errors_exit_one():
    assert run_cli("--nx", "0", "--ny", "2", "--nz", "2").returncode == 1
    assert run_cli("--ny", "2", "--nz", "2").returncode == 1          # --nx missing
    assert run_cli("--nx", "2", "--ny", "2", "--nz", "2", "--procs", "2,1").returncode == 1
    assert run_cli("--nx", "2", "--ny", "2", "--nz", "2", "--cg-tol", "0").returncode == 1


def test_csv_row_per_partition_and_empty_cells(tmp_path):
    for error in (False, True):
        path = tmp_path / f"r{int(error)}.csv"
        RB.emit_report(_synthetic_report(error), "csv", path)
        rows = list(csv.DictReader(path.open()))
        assert [r["partition"] for r in rows] == ["0", "1"]
        assert list(rows[0]) == list(RB.CSV_RUN_COLUMNS + RB.CSV_PARTITION_COLUMNS)
        if error:
            assert all(r["spmv_ratio"] == "" and r["optimized_spmv_seconds"] == "" for r in rows)
            assert all(r["error"] == "DiaFillOverflow" for r in rows)
        else:
            assert rows[0]["spmv_ratio"] == "2.0" and rows[0]["validation_passed"] == "true"


def test_json_roundtrip_and_stdout(tmp_path, capsys):
    rep = _synthetic_report()
    RB.emit_report(rep, "json", tmp_path / "r.json")
    assert json.loads((tmp_path / "r.json").read_text()) == rep.to_dict()
    RB.emit_report(rep, "json", None)
    assert json.loads(capsys.readouterr().out) == rep.to_dict()
    with pytest.raises(ValueError):
        RB.emit_report(rep, "xml", None)


# ----------------------------------------------------------------- device --

gpu = pytest.mark.gpu


def small(**kw):
    base = dict(nx=4, ny=4, nz=4, iters=5, reps=2)
    base.update(kw)
    return ds.BenchConfig(**base)


@gpu
def test_run_benchmark_happy_path():
    d = ds.run_benchmark(small(cg_max_iters=100)).to_dict()
    assert d["error"] is None and d["validation"]["passed"] is True
    assert d["reference_spmv_seconds"] > 0 and d["optimized_spmv_seconds"] > 0
    assert d["spmv_ratio"] == pytest.approx(d["reference_spmv_seconds"]
                                            / d["optimized_spmv_seconds"])
    assert d["cg_seconds"] > 0 and d["cg_converged"] is True
    assert len(d["partitions"]) == 1
    assert "remote part is empty on every partition" in d["notes"]
    assert d["device"]["optimized"]["gflops"] > 0


@gpu
def test_format_flags_and_tuned_multi():
    part = ds.run_benchmark(small(local_format=ds.FormatId.DIA)).to_dict()["partitions"][0]
    assert (part["local_format"], part["remote_format"], part["remote_empty"]) == \
        ("dia", "csr", True)
    d = ds.run_benchmark(small(procs=(2, 1, 1), tune=True, mode="multi")).to_dict()
    assert d["error"] is None and len(d["partitions"]) == 2
    for p in d["partitions"]:
        assert p["local_format"] in ("coo", "csr", "dia")
        assert p["remote_format"] in ("coo", "csr")   # the remote part overflows DIA


@gpu
def test_conversion_failure_yields_partial_report():
    d = ds.run_benchmark(small(nx=8, ny=8, nz=8, procs=(2, 1, 1),
                               remote_format=ds.FormatId.DIA)).to_dict()
    assert d["error"]["phase"] == "optimization_setup"
    assert d["error"]["remote_format"] == "dia"
    assert d["validation"] is None and d["optimized_spmv_seconds"] is None
    assert d["spmv_ratio"] is None and d["reference_spmv_seconds"] > 0


@gpu
def test_validation_failure_blocks_optimized_timing_and_exits_two(monkeypatch, capsys):
    def failing(backend, problem, splits):
        raise ds.ValidationFailed("forced", report=ValidationReport(
            passed=False, converged=False, iterations=50, iteration_bound=12,
            final_residual=1.0))
    monkeypatch.setattr(RB, "validate_solver", failing)
    d = ds.run_benchmark(small()).to_dict()
    assert d["validation"]["passed"] is False
    assert d["optimized_spmv_seconds"] is None and d["spmv_ratio"] is None
    assert RB.main(["--nx", "2", "--ny", "2", "--nz", "2", "--iters", "2"]) == 2
    capsys.readouterr()


@gpu
def test_cli_runs(tmp_path):
    out = tmp_path / "run.json"
    proc = run_cli("--nx", "16", "--ny", "16", "--nz", "16", "--local-format", "dia",
                   "--iters", "30", "--cg-max-iters", "200", "--output", str(out))
    assert proc.returncode == 0, proc.stderr
    rep = json.loads(out.read_text())
    assert rep["validation"]["passed"] is True and rep["spmv_ratio"] is not None
    assert rep["partitions"][0]["remote_empty"] is True and rep["cg_converged"] is True
    out = tmp_path / "multi.csv"
    proc = run_cli("--nx", "4", "--ny", "4", "--nz", "4", "--procs", "2,1,1", "--mode",
                   "multi", "--tune", "--reps", "3", "--iters", "10", "--format", "csv",
                   "--output", str(out))
    assert proc.returncode == 0, proc.stderr
    rows = list(csv.DictReader(out.open()))
    assert len(rows) == 2 and all(r["mode"] == "multi" for r in rows)
