"""bench.py keeps the driver's contract: one JSON line with the required keys
(the reference arm runs on the CPU here; our arm needs the B200)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout,
                       env=dict(os.environ, OPENBLAS_NUM_THREADS="2"))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "3", "--nx", "16"])
    assert d["impl"] == "reference" and BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["higher_is_better"] is True and d["unit"] == "GFLOP/s"
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("hpcg_cg_27pt_")


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--steps", "20", "--warmup", "10", "--nx", "32", "--no-cpu", "--no-sweep",
              "--no-config5", "--no-mg", "--no-powerlaw"])
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 1 and d["steps"] == 20
    assert d["value"] > 0 and d["dtype"] == "f64" and d["scaling"] == "weak"
    roof = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(roof)
    assert roof["bound"] == "hbm" and 0 < roof["frac"] < 1.5
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"]
    assert d["cg_state"]["iter"] == 30 and d["cg_state"]["done"] == 0
