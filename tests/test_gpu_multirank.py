"""GPU: the one-partition-per-process CG (dist.RankCG) at world sizes 2, 4
and 8 -- the procs of BASELINE config 3 -- against the oracle's distributed
CG (reference solver.py:120-189, stencil.py:280-319).

A single B200 is enough: every rank is a process on cuda:0 and the peer
transport's CUDA-IPC mappings alias the same HBM, so the exchange code
(push into the neighbour's ghost slots, flags, the rank-ordered dot
all-gather) runs exactly as it does across an NVSwitch node -- only the
timing differs.  The ranks' contexts time-slice, so the waits use the
stream-memop mode (no SM held while blocked).  On a multi-GPU box the same
worker spreads the ranks over the GPUs.
"""

from __future__ import annotations

import os
import signal
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
from oracle import dynsparse_oracle as O  # noqa: E402


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_ranks(tmp_path, grid, procs, *, local_format="dia", transport="peer", wait="memop",
              tune=False, graph_steps=1, tol=1e-9, timeout=600):
    world = procs[0] * procs[1] * procs[2]
    env = dict(os.environ, DS_PEER_WAIT=wait, OMP_NUM_THREADS="1",
               OPENBLAS_NUM_THREADS="1", PYTHONPATH=ROOT)
    import torch
    if transport == "nccl" and torch.cuda.device_count() < world:
        env["DS_TEST_NCCL_FAKE_HOSTS"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.join(ROOT, "tests", "mp_rank_worker.py"),
           "--grid", *map(str, grid), "--procs", *map(str, procs),
           "--local-format", local_format, "--transport", transport, "--tol", str(tol),
           "--graph-steps", str(graph_steps), "--out", str(tmp_path)]
    if tune:
        cmd.append("--tune")
    # own process group: a timeout kills the launcher AND every rank (a rank
    # left blocked on a flag would otherwise keep its context on the GPU)
    proc = subprocess.Popen(cmd, env=env, cwd=ROOT, stdout=subprocess.PIPE,
                            stderr=subprocess.PIPE, text=True, start_new_session=True)
    try:
        out_s, err_s = proc.communicate(timeout=timeout)
    except subprocess.TimeoutExpired:
        os.killpg(proc.pid, signal.SIGKILL)
        out_s, err_s = proc.communicate()
        pytest.fail(f"ranks timed out after {timeout} s: {err_s[-4000:]}")
    assert proc.returncode == 0, out_s[-3000:] + err_s[-6000:]
    out = []
    for r in range(world):
        with np.load(os.path.join(tmp_path, f"rank{r}.npz")) as z:
            out.append({k: z[k] for k in z.files})
    return out


def oracle_dist(grid, procs, tol=1e-9):
    parts = O.stencil_problem(*grid, *procs)
    splits = [O.split(p) for p in parts]
    return O.cg_dist(parts, splits, [p.b for p in parts], tol=tol)


def check_against_oracle(outs, ref):
    its = {int(o["iterations"]) for o in outs}
    assert len(its) == 1, f"ranks disagree on the iteration count: {its}"
    it = its.pop()
    assert abs(it - ref.iterations) <= 1       # reference test_solver.py:121
    for o in outs[1:]:                          # every rank holds the same history bits
        assert o["history"].tobytes() == outs[0]["history"].tobytes()
    hist = outs[0]["history"]
    k = min(it, ref.iterations) + 1
    assert np.all(np.abs(hist[:k] - ref.history[:k]) <= 1e-8 * ref.history[:k] + 1e-14)
    for r, o in enumerate(outs):
        assert bool(o["converged"])
        assert np.max(np.abs(o["x"] - ref.x[r])) < 1e-8
        assert np.max(np.abs(o["x"] - 1.0)) < 1e-6    # xexact = 1 (test_solver.py:78-83)


@pytest.mark.parametrize("procs", [(2, 1, 1), (2, 2, 1), (2, 2, 2)])
def test_peer_rank_cg_matches_oracle(tmp_path, procs):
    grid = (10, 8, 6)
    outs = run_ranks(tmp_path, grid, procs)
    check_against_oracle(outs, oracle_dist(grid, procs))


def test_peer_rank_cg_csr_local_graph_chunks(tmp_path):
    """CSR local parts and 5 iterations per captured graph (the bench's
    replay pattern): converged no-op steps still exchange, ranks stay in step."""
    grid, procs = (8, 8, 8), (2, 2, 2)
    outs = run_ranks(tmp_path, grid, procs, local_format="csr", graph_steps=5)
    check_against_oracle(outs, oracle_dist(grid, procs))


def test_peer_spin_wait_two_ranks(tmp_path):
    """The in-kernel spin wait (the multi-GPU default) with two ranks time-
    slicing one GPU: slower, but it must complete and match."""
    grid, procs = (8, 6, 4), (2, 1, 1)
    outs = run_ranks(tmp_path, grid, procs, wait="spin", timeout=900)
    check_against_oracle(outs, oracle_dist(grid, procs))


def test_tuner_modes_agree_across_ranks(tmp_path):
    """select_rank_plan: morpheus / ghost are one format on every rank (the
    all-reduce MAX across processes); multi is rank-local."""
    grid, procs = (12, 10, 8), (2, 2, 1)
    outs = run_ranks(tmp_path, grid, procs, tune=True)
    plans = np.stack([o["plans"] for o in outs])        # (ranks, 4 modes, 2)
    for m in (1, 2, 3):                                 # morpheus, ghost, morpheus amortised
        assert (plans[:, m] == plans[0, m]).all(), plans[:, m]
    csr = 1
    assert (plans[:, 1, 1] == csr).all() and (plans[:, 2, 0] == csr).all()
    assert (plans[:, 2, 1] != 2).all()       # the remote part overflows DIA: never chosen
    check_against_oracle(outs, oracle_dist(grid, procs))


@pytest.mark.timeout(420)
@pytest.mark.skipif(os.environ.get("DS_TEST_NCCL_ONE_GPU") != "1",
                    reason="NCCL ranks sharing one GPU talk over sockets and spin while their "
                           "contexts time-slice (minutes); opt in with DS_TEST_NCCL_ONE_GPU=1 "
                           "or run on a multi-GPU node")
def test_nccl_rank_cg_matches_oracle(tmp_path):
    """The NCCL transport (pack kernels + grouped send/recv + ncclAllGather)
    at world 2.  On one GPU the ranks claim distinct NCCL host ids and talk
    over NCCL's socket transport (slow: NCCL's kernels spin while the two
    contexts time-slice); on a node they use NVLink."""
    grid, procs = (6, 4, 4), (2, 1, 1)
    outs = run_ranks(tmp_path, grid, procs, transport="nccl", timeout=400)
    check_against_oracle(outs, oracle_dist(grid, procs))


@pytest.mark.parametrize("procs", [(2, 1, 1), (2, 2, 1), (2, 2, 2)])
def test_peer_rank_cg_matches_reference_golden(tmp_path, procs):
    """16^3 per rank on the bench's process grids against the REFERENCE's own
    distributed CG (tests/golden/cgdist16.npz from make_golden.py)."""
    from conftest import GOLDEN
    with np.load(os.path.join(GOLDEN, "cgdist16.npz")) as z:
        key = "p%d%d%d" % procs
        ref = type("Ref", (), {})()
        ref.iterations = int(z[f"{key}/iterations"])
        ref.history = z[f"{key}/history"]
        ref.x = [z[f"{key}/x{k}"] for k in range(procs[0] * procs[1] * procs[2])]
    outs = run_ranks(tmp_path, (16, 16, 16), procs, graph_steps=4)
    check_against_oracle(outs, ref)


def test_peer_rank_cg_40_cubed_two_ranks(tmp_path):
    """40^3 per rank: the DIA pipeline's grid exceeds 128 CTAs (the fused,
    ticket-completed partition p.Ap must see every CTA's partial)."""
    grid, procs = (40, 40, 40), (2, 1, 1)
    outs = run_ranks(tmp_path, grid, procs, graph_steps=5)
    check_against_oracle(outs, oracle_dist(grid, procs))
