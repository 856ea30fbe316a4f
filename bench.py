#!/usr/bin/env python
"""bench.py -- HPCG-style CG on B200 (BASELINE.json metric: "SpMV GFLOP/s & HBM
GB/s per format; HPCG CG GFLOP/s at 1/2/4/8 B200").

A "step" is ONE conjugate-gradient iteration (solver.py:170-188) on a 27-point
stencil with a 104^3 local grid per GPU (BASELINE config 3): halo exchange,
SpMV (local part DIA, remote part CSR -- the paper's multi-format plan), the
two global dots, three WAXPBY-equivalent updates.  Flops per step are HPCG's
2*nnz + 10*n.  GPUs -> process grid (1,1,1) (2,1,1) (2,2,1)
(2,2,2); one process per GPU, weak scaling.

Printed JSON (rank 0, one line): value = whole-job GFLOP/s of the K timed
steps (CUDA events, max over ranks), plus
  spmv_sweep  -- config 2: COO / CSR / DIA SpMV at 104^3 (GFLOP/s, GB/s, frac)
  powerlaw    -- config 4: irregular ~54.5M-nnz matrix, CSR vs COO (+ DIA
                 overflow), conversion time, the tuner's pick
  roofline    -- the dominant kernel (fused DIA SpMV + p.Ap) of the CG step
  e2e         -- the same metric through the public API with host buffers
  cpu_baseline-- the CPU oracle (oracle/, numpy port of the reference) timed
                 on this host's cores on a bounded sample
  clocks      -- nvidia-smi samples taken during the measurements

``--impl reference`` times the reference's CPU implementation (the oracle
port; the reference itself is pure Python and cannot travel to the box) on
the same config, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

PROCS = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}
METRIC = "HPCG CG GFLOP/s (27-pt stencil, 104^3 per GPU)"


def procs_for(n: int) -> tuple[int, int, int]:
    if n in PROCS:
        return PROCS[n]
    raise SystemExit(f"unsupported GPU count {n} (use 1, 2, 4 or 8)")


def measured_traffic(kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the latest
    committed ncu capture (profiles/r02/traffic.json, else r01), or None."""
    for rnd in ("r02", "r01"):
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "traffic.json")) as fh:
                return int(json.load(fh)[kernel]["dram_bytes_per_launch"])
        except Exception:
            continue
    return None


def peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return {"hbm_gbs": float(p["hbm_gbs"]), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback"}


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the measurements)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if s > 0.5 * mx] if mx else []
        return {"sm_mhz": statistics.median(loaded) if loaded else (statistics.median(sm) if sm else None),
                "sm_max_mhz": mx or None, "reasons": sorted(reasons), "samples": len(sm),
                "samples_under_load": len(loaded)}


# ---------------------------------------------------------------------------
# problem setup
# ---------------------------------------------------------------------------

def flops_per_iter(nnz: int, n: int) -> int:
    return 2 * nnz + 10 * n


def dia_bytes(n: int, ncols: int, ndiags: int) -> int:
    return 8 * ndiags * n + 8 * ndiags + 8 * ncols + 8 * n


def csr_bytes(n: int, ncols: int, nnz: int) -> int:
    return 12 * nnz + 4 * (n + 1) + 8 * ncols + 8 * n


def coo_bytes(n: int, ncols: int, nnz: int) -> int:
    return 16 * nnz + 8 * ncols + 8 * n


def format_array_bytes(fmt: str, n: int, nnz: int, ndiags: int) -> int:
    """Bytes of a matrix's arrays (int32 indices, f64 values)."""
    if fmt == "csr":
        return 4 * (n + 1) + 12 * nnz
    if fmt == "coo":
        return 16 * nnz
    return 8 * n * ndiags + 4 * ndiags


def convert_floor(pairs_ms: dict, n: int, nnz: int, ndiags: int, peak_gbs: float) -> dict:
    """Each conversion against its byte floor: the source's arrays read once
    and the target's written once at the measured copy bandwidth."""
    out = {}
    for pair, ms in pairs_ms.items():
        a, b = pair.split("->")
        by = format_array_bytes(a, n, nnz, ndiags) + format_array_bytes(b, n, nnz, ndiags)
        floor_ms = by / (peak_gbs * 1e9) * 1e3
        out[pair] = {"bytes": by, "floor_ms": round(floor_ms, 3), "frac": round(floor_ms / ms, 3)}
    return out


def build_rank(ds, spec, rank, dev, local_fmt, remote_fmt):
    """This rank's partition on the device, split and converted (host setup)."""
    part = ds.generate_partition(spec, rank, space=ds.MemorySpace.DEVICE, device=dev)
    prob = ds.PartitionedProblem(spec, [part])
    split = ds.split_local_remote(prob, 0)
    ds.convert_inplace(split.local, local_fmt)
    try:
        ds.convert_inplace(split.remote, remote_fmt)
    except ds.DiaFillOverflow:
        pass  # remote DIA overflows on the stencil: keep CSR like the tuner's skip
    return part, split


# ---------------------------------------------------------------------------
# SpMV sweeps (config 2 and 4)
# ---------------------------------------------------------------------------

def time_spmv(ds, torch, m, x, y, warm=20, reps=200, batch=40):
    """Per-launch time (ms) of y = A x: CUDA events on the launch stream
    around batches of back-to-back launches (prepared launchers: one ctypes
    call of host time each, so the device never waits for Python), median
    over the batches."""
    from paper_2209_06478_b200.kernels import prepared_spmv
    st = torch.cuda.current_stream()
    launch = prepared_spmv(m, x, y, 0)
    for _ in range(warm):
        launch()
    nb = max(1, reps // batch)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(nb)]
    torch.cuda.synchronize()
    for e0, e1 in ev:
        e0.record(st)
        for _ in range(batch):
            launch()
        e1.record(st)
    torch.cuda.synchronize()
    return statistics.median(e0.elapsed_time(e1) / batch for e0, e1 in ev)


def _gpu_ms(torch, fn, reps: int = 3) -> float:
    """Best-of wall ms of a device operation, CUDA-synchronised on both sides."""
    best = float("inf")
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    return round(best, 3)


def sweep_104(ds, torch, a_full, dev, peak, cpu=None):
    """BASELINE config 2: COO / CSR / DIA SpMV of the 104^3 stencil (median
    per launch), the four conversions between them, and -- with ``cpu`` (the
    oracle's numbers on this host) -- the CPU serial / threaded times beside."""
    import numpy as np
    n = a_full.nrows
    x = ds.DenseVector(torch.from_numpy(np.random.default_rng(0).standard_normal(n)).to(dev))
    y = ds.DenseVector.zeros(n, ds.MemorySpace.DEVICE, dev)
    out = {}
    mats = {}
    for name in ("coo", "csr", "dia"):
        m = ds.convert(a_full, ds.FormatId[name.upper()])
        mats[name] = m
        ms = time_spmv(ds, torch, m, x, y)
        nnz = a_full.nnz
        if name == "csr":
            b = csr_bytes(n, n, nnz)
        elif name == "coo":
            b = coo_bytes(n, n, nnz)
        else:
            b = dia_bytes(n, n, m.ndiags)
        gbs = b / (ms * 1e-3) / 1e9
        out[name] = {"ms": round(ms, 5), "gflops": round(2 * nnz / (ms * 1e-3) / 1e9, 1),
                     "gbs": round(gbs, 1), "frac": round(gbs / peak, 3), "bytes": b}
        if cpu and name in cpu.get("spmv", {}):
            c = cpu["spmv"][name]
            out[name]["cpu_serial_ms"] = c["serial_ms"]
            out[name]["cpu_threaded_ms"] = c["threaded_ms"]
            out[name]["speedup_vs_cpu_threaded"] = round(c["threaded_ms"] / ms, 1)
    F = ds.FormatId
    conv = {"csr->dia": _gpu_ms(torch, lambda: ds.convert(mats["csr"], F.DIA)),
            "dia->csr": _gpu_ms(torch, lambda: ds.convert(mats["dia"], F.CSR)),
            "csr->coo": _gpu_ms(torch, lambda: ds.convert(mats["csr"], F.COO)),
            "coo->csr": _gpu_ms(torch, lambda: ds.convert(mats["coo"], F.CSR))}
    out["convert_ms"] = conv
    out["convert_vs_byte_floor"] = convert_floor(conv, n, a_full.nnz, mats["dia"].ndiags, peak)
    if cpu and "convert_ms" in cpu:
        out["cpu_convert_ms"] = cpu["convert_ms"]
        out["cpu_cores"] = cpu["cores"]
    del mats
    return out


def sweep_powerlaw(ds, torch, dev, peak, cpu_threads: int = 0):
    """BASELINE config 4: generator of BASELINE.md §2, device conversion, CSR vs
    COO SpMV, DIA overflow; the tuner's choice is the measured-fastest format."""
    import numpy as np
    t0 = time.time()
    rng = np.random.default_rng(2209)
    n = 4_194_304
    L = np.minimum(n, np.floor(6.0 * (1.0 - rng.random(n)) ** (-1 / 1.8))).astype(np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), L)
    cols = rng.integers(0, n, rows.size)
    vals = rng.standard_normal(rows.size)
    gen_s = time.time() - t0
    # the first conversions pay lazy kernel loading and memory-pool growth:
    # report the fastest of three, each from a fresh raw COO (no cached plan)
    conv_all = []
    for rep in range(3):
        coo = ds.CooMatrix(n, n, rows, cols, vals, ds.MemorySpace.DEVICE, dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        csr = ds.convert(coo, ds.FormatId.CSR)
        torch.cuda.synchronize()
        conv_all.append((time.perf_counter() - t0) * 1e3)
        del coo
    conv_ms = min(conv_all)
    del rows, cols, vals
    ccoo = ds.convert(csr, ds.FormatId.COO)
    nnz = csr.nnz
    x = ds.DenseVector(torch.from_numpy(np.random.default_rng(1).standard_normal(n)).to(dev))
    y = ds.DenseVector.zeros(n, ds.MemorySpace.DEVICE, dev)
    out = {"nnz": nnz, "host_generate_s": round(gen_s, 2), "convert_coo_to_csr_ms": round(conv_ms, 2),
           "convert_coo_to_csr_ms_all": [round(t, 2) for t in conv_all]}
    for name, m, b in (("csr", csr, csr_bytes(n, n, nnz)), ("coo", ccoo, coo_bytes(n, n, nnz))):
        ms = time_spmv(ds, torch, m, x, y, warm=10, reps=50)
        gbs = b / (ms * 1e-3) / 1e9
        out[name] = {"ms": round(ms, 4), "gflops": round(2 * nnz / (ms * 1e-3) / 1e9, 1),
                     "gbs": round(gbs, 1), "frac": round(gbs / peak, 3)}
    # the random-gather floor measured on this GPU in this run: the CSR
    # SpMV's column + value stream and x gathers without the row structure
    # (ds_probe_gather); the SpMVs are reported against it too
    from paper_2209_06478_b200 import _native
    lib = _native.load()
    sink = torch.zeros(1, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev)
    probe = lambda: _native.check(lib.ds_probe_gather(  # noqa: E731
        nnz, csr.col_indices.data_ptr(), csr.values.data_ptr(), x.data.data_ptr(),
        sink.data_ptr(), st.cuda_stream))
    for _ in range(5):
        probe()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        probe()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    floor_ms = statistics.median(ts)
    out["gather_floor"] = {
        "ms": round(floor_ms, 4), "gathers_per_s": round(nnz / (floor_ms * 1e-3), 0),
        "hbm_frac_ceiling_csr": round(csr_bytes(n, n, nnz) / (floor_ms * 1e-3) / 1e9 / peak, 3),
        "what": "ds_probe_gather: stream cols + values, gather x[col] (no rows); every 8-B "
                "random gather costs one L1 tag request, which bounds the irregular SpMV"}
    for name in ("csr", "coo"):
        out[name]["frac_of_gather_floor"] = round(floor_ms / out[name]["ms"], 3)
    if cpu_threads:
        a_host = (n, csr.row_offsets.cpu().numpy(), csr.col_indices.cpu().numpy(),
                  csr.values.cpu().numpy())
        c = cpu_formats_sample(a_host, cpu_threads, convert=False)["spmv"]
        for name in ("csr", "coo"):
            out[name]["cpu_serial_ms"] = c[name]["serial_ms"]
            out[name]["cpu_threaded_ms"] = c[name]["threaded_ms"]
            out[name]["speedup_vs_cpu_threaded"] = round(c[name]["threaded_ms"] / out[name]["ms"], 1)
        out["cpu_cores"] = cpu_threads
    try:
        ds.convert(csr, ds.FormatId.DIA)
        out["dia"] = "converted"
    except ds.DiaFillOverflow as exc:
        out["dia"] = f"DiaFillOverflow: {str(exc)[:60]}"
    out["selected"] = min(("csr", "coo"), key=lambda k: out[k]["ms"])
    return out


def format_switching(ds, torch, dev, peak, nx: int = 192, steps: int = 100) -> dict:
    """BASELINE config 5 on this GPU: a 192^3 local grid, the per-GPU tuner
    ('multi': every (local, remote) combination converted in place -- the
    runtime switching cost -- and timed), the chosen plan applied, then
    ``steps`` graph-replayed CG iterations.  Reports the conversion cost in
    SpMV-equivalents and the CG rate with and without it."""
    from paper_2209_06478_b200 import dist as D
    from paper_2209_06478_b200 import solver as S
    spec = ds.GridSpec(nx, nx, nx)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    part = ds.generate_partition(spec, 0, space=ds.MemorySpace.DEVICE, device=dev)
    split = ds.split_local_remote(ds.PartitionedProblem(spec, [part]), 0)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    prof = D.profile_rank(part, split, reps=5)
    # the pick pays each combination's measured switch cost amortised over
    # the planned iterations ("format switching with conversion cost included")
    lf, rf = D.select_rank_plan(prof["entries"], "multi", 1, prof["convert_s"], steps)
    lf0, rf0 = D.select_rank_plan(prof["entries"], "multi", 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ds.convert_inplace(split.local, lf)
    ds.convert_inplace(split.remote, rf)
    torch.cuda.synchronize()
    conv_ms = (time.perf_counter() - t0) * 1e3
    n, nnz = part.a_full.nrows, part.a_full.nnz
    eng, _ = S.build_engine(S.DistributedOperator(ds.PartitionedProblem(spec, [part]), [split]),
                            [part.b], None, 1e-300, steps + 32)
    st = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        eng.setup(st.cuda_stream)
        eng.capture_step(10)          # 10 iterations per graph replay
        eng.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps // 10):
            eng.replay()
        e1.record(st)
        torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / steps
    fl = flops_per_iter(nnz, n)
    spmv_ms = prof["entries"][(lf, rf)] * 1e3
    out = {
        "grid": [nx, nx, nx], "n": n, "nnz": nnz, "generate_on_device_s": round(gen_s, 3),
        "plan": [lf.name.lower(), rf.name.lower()],
        "plan_ignoring_switch_cost": [lf0.name.lower(), rf0.name.lower()],
        "selection": f"tuner multi, switch cost amortised over {steps} iterations",
        "spmv_us": {f"{a.name.lower()}/{b.name.lower()}": round(t * 1e6, 1)
                    for (a, b), t in sorted(prof["entries"].items())},
        "convert_from_csr_ms": {f"{a.name.lower()}/{b.name.lower()}": round(t * 1e3, 3)
                                for (a, b), t in sorted(prof["convert_s"].items())},
        "apply_convert_ms": round(conv_ms, 3),
        "convert_in_spmv_equivalents": round(conv_ms / spmv_ms, 1),
        "cg_ms_per_step": round(step_ms, 4),
        "cg_gflops": round(fl / (step_ms * 1e-3) / 1e9, 1),
        "cg_gflops_incl_conversion": round(steps * fl / ((steps * step_ms + conv_ms) * 1e-3) / 1e9, 1),
        "steps": steps,
    }
    del eng, split, part
    torch.cuda.empty_cache()
    return out


def hpcg_mg(ds, torch, dev, nx: int = 104, iters: int = 50) -> dict:
    """HPCG proper on this GPU (north star: "HPCG's dot, WAXPBY and SymGS/MG
    kernels"; the reference stops at plain CG, so parity is against the
    repo's CPU restatement only): 4-level hierarchy, coloured SymGS, one
    PCG iteration = one CUDA graph replay.  Flops per iteration follow HPCG's
    count: SpMV 2 nnz0; per V-cycle level above the coarsest pre-/post-SymGS
    4 nnz_l each + the residual SpMV 2 nnz_l; the coarsest one SymGS 4 nnz_L;
    3 dots and 3 WAXPBY 2n each."""
    from paper_2209_06478_b200 import hpcg
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = hpcg.MgHierarchy.build(nx, nx, nx, device=dev)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    part = ds.generate_partition(ds.GridSpec(nx, nx, nx), 0, space=ds.MemorySpace.DEVICE,
                                 device=dev)
    nnz = [L.a.nnz for L in h.levels]
    n0 = h.levels[0].nrows
    fl = 2 * nnz[0] + sum(10 * z for z in nnz[:-1]) + 4 * nnz[-1] + 12 * n0
    # convergence: a solve to 1e-9 capped at HPCG's 50 iterations per set (the
    # injection-restriction V-cycle's count grows with the grid: 15 at 16^3,
    # 26 at 32^3 in the CPU restatement; 104^3 stops at the cap)
    res = hpcg.pcg(h, part.b, tol=1e-9, max_iters=iters)
    eng = hpcg.PcgEngine(h, part.b, tol=0.0, max_iters=10**6)
    eng.setup()
    eng._capture(1)
    for _ in range(3):
        eng.graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        eng.graph.replay()
    e1.record()
    torch.cuda.synchronize()
    it_ms = e0.elapsed_time(e1) / iters
    out = {"grid": [nx, nx, nx], "levels": [L.nrows for L in h.levels], "nnz_per_level": nnz,
           "build_s": round(build_s, 3), "ms_per_iteration": round(it_ms, 4),
           "gflops": round(fl / (it_ms * 1e-3) / 1e9, 1), "flops_per_iteration": fl,
           "iterations_to_1e-9": int(res.iterations), "converged": bool(res.converged),
           "relative_residual": float(res.residual_history[-1]),
           "parity": "bitwise SymGS / V-cycle vs the CPU restatement (tests/test_gpu_hpcg.py); "
                     "no reference implementation exists (SURVEY 8f)"}
    del eng, h
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# CPU baseline (oracle port of the reference), bounded sample
# ---------------------------------------------------------------------------

def cpu_cg_sample(spec_args, iters: int, threads: int, local_fmt: str = "csr") -> dict:
    """Time ``iters`` CG iterations of the oracle on the host (untimed setup),
    the reference's own loop (solver.py:170-188) with its threaded backend.
    The local part runs in ``local_fmt`` -- CSR by default, the CPU's fastest
    format with threads; the remote part is CSR."""
    import numpy as np
    from oracle import dynsparse_oracle as O
    nx, ny, nz, px, py, pz = spec_args
    parts = [O.stencil_partition(nx, ny, nz, px, py, pz, r) for r in range(px * py * pz)]
    fmt = {"coo": O.COO, "csr": O.CSR, "dia": O.DIA}[local_fmt]
    splits = []
    for p in parts:
        loc, rem = O.split(p)
        splits.append((loc if fmt == O.CSR else O.convert(loc, fmt), rem))
    P = len(parts)
    n = parts[0].a_full.nrows
    bs = [p.b for p in parts]
    # one untimed setup, then time the loop body
    x = [np.zeros(n) for _ in range(P)]
    p_full = [np.zeros(n + parts[k].ghost_count) for k in range(P)]
    p = [pf[:n] for pf in p_full]
    r = [b.copy() for b in bs]
    ap = [np.zeros(n) for _ in range(P)]
    for k in range(P):
        p[k][:] = r[k]
    rr = sum(O.dot(r[k], r[k]) for k in range(P))
    nnz_total = sum(p.a_full.vals.size for p in parts)
    t0 = time.perf_counter()
    for _ in range(iters):
        O.dist_spmv(parts, splits, p_full, ap, nthreads=threads)
        pap = sum(O.dot(p[k], ap[k]) for k in range(P))
        alpha = rr / pap
        for k in range(P):
            O.waxpby(1.0, x[k], alpha, p[k], x[k])
            O.waxpby(1.0, r[k], -alpha, ap[k], r[k])
        rr_new = sum(O.dot(r[k], r[k]) for k in range(P))
        beta = rr_new / rr
        for k in range(P):
            O.waxpby(1.0, r[k], beta, p[k], p[k])
        rr = rr_new
    dt = time.perf_counter() - t0
    fl = iters * flops_per_iter(nnz_total, n * P)
    return {"value": round(fl / dt / 1e9, 4), "unit": "GFLOP/s", "cores": threads,
            "kind": "port", "seconds": round(dt, 3),
            "sample": f"{iters} CG iterations of the oracle (numpy port of the reference), "
                      f"grid {nx}^3 x {P} partition(s), local {local_fmt.upper()} + remote CSR, "
                      f"ExecBackend.threaded({threads}), OPENBLAS_NUM_THREADS="
                      f"{os.environ.get('OPENBLAS_NUM_THREADS')}"}


def _best_ms(fn, reps: int) -> float:
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    return round(best, 2)


def cpu_formats_sample(a_host, threads: int, convert: bool = True) -> dict:
    """BASELINE.md §3's CPU rows on the oracle: per-format SpMV serial and
    threaded(N) (kernels.py:102-163) and, with ``convert``, the conversions
    CSR<->DIA and CSR<->COO (datamove.py:261-281); best-of wall ms.
    ``a_host`` = (nrows, offsets, cols, vals) of a canonical CSR."""
    import numpy as np
    from oracle import dynsparse_oracle as O
    n, off, cols, vals = a_host
    a = O.csr(n, n, off.astype(np.int64), cols.astype(np.int64), vals)
    out = {"cores": threads, "kind": "port"}
    mats = {"csr": a}
    if convert:
        conv = {}
        t0 = time.perf_counter()
        mats["dia"] = O.convert(a, O.DIA)
        conv["csr->dia"] = round((time.perf_counter() - t0) * 1e3, 1)
        conv["dia->csr"] = _best_ms(lambda: O.convert(mats["dia"], O.CSR), 1)
        t0 = time.perf_counter()
        mats["coo"] = O.convert(a, O.COO)
        conv["csr->coo"] = round((time.perf_counter() - t0) * 1e3, 1)
        conv["coo->csr"] = _best_ms(lambda: O.convert(mats["coo"], O.CSR), 1)
        out["convert_ms"] = conv
    else:   # the canonical COO of a canonical CSR: its rows expanded
        mats["coo"] = O.coo(n, n, np.repeat(np.arange(n, dtype=np.int64), np.diff(a.offsets)),
                            a.cols, a.vals)
    x = np.random.default_rng(0).standard_normal(n)
    y = np.zeros(n)
    spmv = {}
    for name in ("coo", "csr", "dia"):
        if name not in mats:
            continue
        m = mats[name]
        spmv[name] = {"serial_ms": _best_ms(lambda: O.spmv(m, x, y, 1), 2),
                      "threaded_ms": _best_ms(lambda: O.spmv(m, x, y, threads), 3)}
    out["spmv"] = spmv
    return out


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def config_of(nx: int, px: int, py: int, pz: int) -> dict:
    """The workload both arms run (the per-arm format plan is reported apart)."""
    return {"workload": f"hpcg_cg_27pt_{nx}^3_per_gpu", "grid_per_gpu": [nx, nx, nx],
            "procs": [px, py, pz], "tol_timed": "1e-300 (fixed step count)",
            "l2": (f"no flush: the matrix ({8 * 27 * nx ** 3 / 1e6:.0f} MB/GPU as DIA) exceeds "
                   f"the 126 MB L2 and is re-streamed every step") if 8 * 27 * nx ** 3 > 126e6
            else (f"no flush; the matrix ({8 * 27 * nx ** 3 / 1e6:.0f} MB/GPU as DIA) fits the "
                  f"126 MB L2 -- a test size, not a bench configuration")}


def reference_arm(args, rank: int, world: int) -> int:
    if rank != 0:
        return 0
    threads = host_threads()
    os.environ["OPENBLAS_NUM_THREADS"] = str(threads)
    px, py, pz = procs_for(args.gpus)
    nx = args.nx
    # bounded sample: enough iterations for ~10-60 s of CPU work
    iters = max(1, min(args.steps, 10 if world == 1 else 3))
    res = cpu_cg_sample((nx, nx, nx, px, py, pz), iters, threads, "csr")
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(res["seconds"] / iters * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(nx, px, py, pz),
        "plan": {"local_format": "csr", "remote_format": "csr",
                 "why": "CSR is the CPU's fastest local format with threads (BASELINE.md §3)"},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run(args, rank: int, world: int) -> int:
    import numpy as np
    import torch

    import paper_2209_06478_b200 as ds
    from paper_2209_06478_b200 import solver as S

    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # DS_BENCH_SAME_GPU=1: every rank on cuda:0 (exercises the N > 1 path on a
    # one-GPU box: IPC peer memory between the ranks' contexts, gloo for the
    # host-side collectives, stream-memop waits since the contexts time-slice)
    same_gpu = world > 1 and os.environ.get("DS_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local_rank = 0
        os.environ.setdefault("DS_PEER_WAIT", "memop")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    pk = peaks()
    peak = pk["hbm_gbs"]
    px, py, pz = procs_for(world)
    nx = args.nx
    spec = ds.GridSpec(nx, nx, nx, px, py, pz)
    clocks = ClockSampler(local_rank)
    clocks.start()

    extras = {}
    if args.fixed_plan:
        part, split = build_rank(ds, spec, rank, dev, ds.FormatId.DIA, ds.FormatId.CSR)
        plan = ("dia", "csr")
    else:
        # dynamic per-GPU format selection (tuner 'multi' on this rank's
        # partition; conversion cost of every switch recorded)
        from paper_2209_06478_b200 import dist as D
        part = ds.generate_partition(spec, rank, space=ds.MemorySpace.DEVICE, device=dev)
        split = ds.split_local_remote(ds.PartitionedProblem(spec, [part]), 0)
        t_tune = time.perf_counter()
        prof = D.profile_rank(part, split, reps=10)
        lf, rf = D.select_rank_plan(prof["entries"], "multi", world)
        t_conv = time.perf_counter()
        ds.convert_inplace(split.local, lf)
        ds.convert_inplace(split.remote, rf)
        torch.cuda.synchronize()
        t_end = time.perf_counter()
        plan = (lf.name.lower(), rf.name.lower())
        extras["tuner"] = {
            "mode": "multi", "plan": list(plan),
            "spmv_us": {f"{a.name.lower()}/{b.name.lower()}": round(t * 1e6, 2)
                        for (a, b), t in sorted(prof["entries"].items())},
            "skipped": [f"{a.name.lower()}/{b.name.lower()}" for a, b in prof["skipped"]],
            "convert_ms": {f"{a.name.lower()}/{b.name.lower()}": round(t * 1e3, 3)
                           for (a, b), t in sorted(prof["convert_s"].items())},
            "tune_s": round(t_conv - t_tune, 3), "apply_convert_ms": round((t_end - t_conv) * 1e3, 3)}
    n = part.a_full.nrows
    nnz_local = part.a_full.nnz
    cpu_fmt = None
    thr = host_threads()
    if world == 1 and rank == 0 and not args.no_cpu:
        # BASELINE.md §3 on this host: the oracle's per-format SpMV (serial /
        # threaded) and conversions at 104^3 (about 20 s of CPU work)
        os.environ["OPENBLAS_NUM_THREADS"] = str(thr)
        a = part.a_full
        cpu_fmt = cpu_formats_sample((n, a.row_offsets.cpu().numpy(), a.col_indices.cpu().numpy(),
                                      a.values.cpu().numpy()), thr)
    if world == 1 and not args.no_sweep:
        extras["spmv_sweep"] = sweep_104(ds, torch, part.a_full, dev, peak, cpu_fmt)
    torch.cuda.synchronize()

    kern_steps = min(args.steps, 200)
    budget = args.warmup + args.steps + kern_steps + 8   # no step may hit max_iters
    if world == 1 and not args.rank_engine:
        eng, _ = S.build_engine(S.DistributedOperator(ds.PartitionedProblem(spec, [part]), [split]),
                                [part.b], None, 1e-300, budget)
    else:
        from paper_2209_06478_b200 import dist as D
        if world == 1 and not torch.distributed.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            torch.distributed.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        eng = D.RankCG(spec, part, split, dev, 1e-300, budget, transport=args.transport)
    st = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        eng.setup(st.cuda_stream)
        use_graph = not args.eager
        # several iterations per graph (fewer graph-launch gaps) when both
        # counts divide; each replay then advances `spg` CG iterations
        spg = 1
        if use_graph:
            for c in (20, 10, 5, 4, 2):
                if args.steps % c == 0 and args.warmup % c == 0:
                    spg = c
                    break
        if use_graph:
            eng.capture_step(spg) if spg > 1 else eng.capture_step()
        step = eng.replay if use_graph else (lambda: eng.step(st.cuda_stream))
        for _ in range(args.warmup // spg):
            step()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.steps // spg):
            step()
        e1.record(st)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        ms = e0.elapsed_time(e1)
        sc = eng.scalars()
        state = {"iter": int(sc.iter), "done": int(sc.done)}

        # dominant kernel: time the fused DIA SpMV launches inside eager steps
        kern = None
        if hasattr(eng, "time_spmv_in_graph") and not args.eager:
            kern = eng.time_spmv_in_graph(kern_steps)
        if kern is None:
            kern = eng.time_spmv_in_steps(kern_steps, st.cuda_stream)
            kern["method"] = "eager steps, CUDA events around the SpMV launch"
        if int(eng.scalars().done) != 0:
            raise RuntimeError("CG stopped inside the measured steps; timings would be no-ops")
        if hasattr(eng, "release_l2"):
            eng.release_l2(st.cuda_stream)   # later legs get the whole L2 back

    clk = clocks.stop()
    nnz_total, ms_max = nnz_local, ms
    if world > 1:
        t = torch.tensor([ms, float(nnz_local)], dtype=torch.float64, device=dev)
        tmax = t.clone()
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        tsum = t.clone()
        torch.distributed.all_reduce(tsum, op=torch.distributed.ReduceOp.SUM)
        ms_max, nnz_total = float(tmax[0]), int(tsum[1])
    fl = args.steps * flops_per_iter(nnz_total, n * world)
    value = fl / (ms_max * 1e-3) / 1e9

    # roofline of the dominant kernel (per launch, algorithmic bytes)
    lm = eng.local if hasattr(eng, "local") else eng.parts[0].local
    if isinstance(lm, ds.DiaMatrix):
        kb = dia_bytes(n, n, lm.ndiags)
    elif isinstance(lm, ds.CsrMatrix):
        kb = csr_bytes(n, n, lm.nnz)
    else:
        kb = coo_bytes(n, n, lm.nnz)
    k_ach = kb / (kern["avg_ms"] * 1e-3) / 1e9 if kern["avg_ms"] > 0 else 0.0
    roof = {"kernel": f"{plan[0]} SpMV of the CG step (fused p.Ap)", "bound": "hbm",
            "achieved": round(k_ach, 1), "peak": peak, "unit": "GB/s",
            "frac": round(k_ach / peak, 3), "traffic": measured_traffic("dia_pipe") if plan[0] == "dia" else None,
            "peak_source": pk["source"],
            "algorithmic_bytes_per_launch": kb, "avg_launch_ms": round(kern["avg_ms"], 5),
            "timing": kern.get("method"),
            "share_of_step": round(kern["avg_ms"] / kern["step_ms"], 3) if kern["step_ms"] else None}

    e2e = None
    cpu = None
    parity = None
    if world > 1 or args.rank_engine:
        e2e = measure_e2e_ranks(torch, eng, part, n, nnz_total, world)
        if world > 1:
            parity = parity_ranks(ds, torch, dev, world, rank, args.transport)
    elif rank == 0:
        e2e = measure_e2e(ds, torch, spec, split, part, n, nnz_local)
    if rank == 0 and world == 1:
        if not args.no_cpu:
            thr = host_threads()
            os.environ["OPENBLAS_NUM_THREADS"] = str(thr)
            cpu = cpu_cg_sample((nx, nx, nx, 1, 1, 1), 60, thr, "csr")   # ~5-10 s of CPU work
            cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
            if cpu_fmt is not None:
                cpu["spmv_104"] = cpu_fmt["spmv"]
                cpu["convert_104_ms"] = cpu_fmt["convert_ms"]
        if not args.no_powerlaw:
            extras["powerlaw"] = sweep_powerlaw(ds, torch, dev, peak,
                                                0 if args.no_cpu else thr)
        if not args.no_config5:
            extras["format_switching_192"] = format_switching(ds, torch, dev, peak)
        if not args.no_mg:
            extras["hpcg_mg"] = hpcg_mg(ds, torch, dev, nx)

    launches_per_step = eng.launches_per_step()
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config_of(nx, px, py, pz),
        "plan": {"local_format": plan[0], "remote_format": plan[1],
                 "format_selection": "fixed" if args.fixed_plan else "tuner multi (per GPU)",
                 "flops_per_step": flops_per_iter(nnz_total, n * world),
                 "graph": not args.eager, "steps_per_graph": spg,
                 "transport": getattr(getattr(eng, "T", None), "name", "in-process")},
        "roofline": roof,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity": parity if parity is not None else (e2e or {}).get("parity"),
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk,
        "cg_state": state,
        "engine": type(eng).__name__ + ("+graph" if getattr(eng, "graph", None) is not None else ""),
        **extras,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()
    return 0


def _golden(name: str) -> dict:
    import numpy as np
    with np.load(os.path.join(ROOT, "tests", "golden", name)) as z:
        return {k: z[k] for k in z.files}


def _history_parity(hist, it, ref_hist, ref_it) -> dict:
    import numpy as np
    k = min(int(it), int(ref_it)) + 1
    rel = float(np.max(np.abs(hist[:k] - ref_hist[:k]) / ref_hist[:k]))
    return {"iterations": int(it), "reference_iterations": int(ref_it),
            "max_history_rel_diff": rel,
            "pass": abs(int(it) - int(ref_it)) <= 1 and rel <= 1e-8}


def parity_ranks(ds, torch, dev, world, rank, transport) -> dict:
    """N > 1: the REFERENCE's distributed CG at 16^3 per rank on this job's
    process grid (tests/golden/cgdist16.npz, written by the real reference
    with tests/golden/make_golden.py) re-run through dist.RankCG with the
    bench's transport; iterations +-1, history within 1e-8, x within 1e-8."""
    import numpy as np
    from paper_2209_06478_b200 import dist as D
    px, py, pz = procs_for(world)
    key = f"p{px}{py}{pz}"
    ref = _golden("cgdist16.npz")
    spec = ds.GridSpec(16, 16, 16, px, py, pz)
    part = ds.generate_partition(spec, rank, space=ds.MemorySpace.DEVICE, device=dev)
    split = ds.split_local_remote(ds.PartitionedProblem(spec, [part]), 0)
    ds.convert_inplace(split.local, ds.FormatId.DIA)
    eng = D.RankCG(spec, part, split, dev, 1e-9, 500, transport=transport)
    try:
        x, it, hist, conv = eng.solve()
    finally:
        eng.close()
    out = _history_parity(hist, it, ref[f"{key}/history"], ref[f"{key}/iterations"])
    xerr = float(np.max(np.abs(x.data.cpu().numpy() - ref[f"{key}/x{rank}"])))
    t = torch.tensor([out["max_history_rel_diff"], xerr, 0.0 if out["pass"] else 1.0],
                     dtype=torch.float64, device=dev)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    out["max_history_rel_diff"], out["max_x_abs_diff_over_ranks"] = float(t[0]), float(t[1])
    out["pass"] = bool(t[2] == 0.0 and t[1] <= 1e-8)
    out.update({"grid_per_rank": [16, 16, 16], "procs": [px, py, pz], "transport": transport,
                "against": "reference golden tests/golden/cgdist16.npz"})
    return out


def measure_e2e(ds, torch, spec, split, part, n, nnz, reps=3):
    """cg() through the public API exactly as a user calls it -- the
    reference's defaults (tol 1e-9, max_iters 500, solver.py:56-70), host
    numpy b in, host numpy x and residual history out, matrix resident on the
    device; wall clock incl. the copies, median of reps; flops = the
    iterations the solve took."""
    import numpy as np
    b_host = ds.DenseVector(part.b.data.cpu().numpy())
    op = ds.DistributedOperator(ds.PartitionedProblem(spec, [part]), [split])
    times, iters = [], 0
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = ds.cg(ds.SERIAL, op, [b_host])
        assert isinstance(res.x[0].data, np.ndarray) and res.converged
        times.append(time.perf_counter() - t0)
        iters = res.iterations
    t = statistics.median(times[1:])
    fl = iters * flops_per_iter(nnz, n)
    out = {"value": round(fl / t / 1e9, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": 8 * n,
           "d2h_bytes_per_step": 8 * n + 8 * (iters + 1),
           "step": f"one ds.cg() solve with the reference's defaults (tol 1e-9): {iters} "
                   f"iterations, host numpy b -> host numpy x",
           "iterations": iters, "seconds": round(t, 5)}
    if spec.nx == 104 and spec.npartitions == 1:
        # the solve's history and x against the REFERENCE's own 104^3 CG
        ref = _golden("cg104.npz")
        par = _history_parity(res.residual_history, res.iterations, ref["history"],
                              ref["iterations"])
        x = res.x[0].data
        par["max_x_sample_abs_diff"] = float(np.max(np.abs(x[::997] - ref["x_sample"])))
        par["pass"] = par["pass"] and par["max_x_sample_abs_diff"] <= 1e-8
        par["against"] = "reference golden tests/golden/cg104.npz"
        out["parity"] = par
    return out


def measure_e2e_ranks(torch, eng, part, n, nnz_total, world, iters=50, reps=3):
    """One partition per process: every rank solves from a host numpy b to a
    host x through its engine (pinned staging, setup, ``iters`` iterations);
    wall time per solve, max over ranks, median of reps."""
    import numpy as np
    b = part.b.data.cpu().numpy() if hasattr(part.b.data, "cpu") else np.asarray(part.b.data)
    times = []
    for _ in range(reps + 1):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x = eng.solve_host(b, iters)
        t = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([t], dtype=torch.float64, device=eng.dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            t = float(tt[0])
        times.append(t)
        assert x.shape == (n,)
    t = statistics.median(times[1:])
    fl = iters * flops_per_iter(nnz_total, n * world)
    return {"value": round(fl / t / 1e9, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": 8 * n,
            "d2h_bytes_per_step": 8 * n,
            "step": f"per rank: host numpy b -> {iters} CG iterations -> host numpy x "
                    f"(dist.RankCG.solve_host), max over {world} rank(s)",
            "seconds": round(t, 5)}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--nx", type=int, default=104)
    ap.add_argument("--eager", action="store_true", help="no CUDA graph for the step")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-powerlaw", action="store_true",
                    help="skip BASELINE config 4 (power-law matrix, ~54.5M nnz)")
    ap.add_argument("--no-mg", action="store_true", help="skip the HPCG multigrid PCG extra")
    ap.add_argument("--no-config5", action="store_true",
                    help="skip BASELINE config 5 (192^3 format switching incl. conversion)")
    ap.add_argument("--fixed-plan", action="store_true",
                    help="local DIA / remote CSR instead of the per-GPU tuner's choice")
    ap.add_argument("--rank-engine", action="store_true",
                    help="at N=1 use the one-partition-per-process engine (dist.RankCG)")
    ap.add_argument("--transport", choices=("peer", "nccl"), default="peer",
                    help="dist.RankCG's halo / dot transport at N > 1 (default: peer memory)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus and args.impl != "reference":
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    return run(args, rank, world)


if __name__ == "__main__":
    sys.exit(main())
