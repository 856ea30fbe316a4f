"""Multi-process (world_size 2, gloo, CPU) checks of the one-partition-per-rank
path.  The device kernels cannot run here, so each rank executes the exact
schedule dist.RankCG issues -- HaloSchedule send/recv pairs, all-gather of
partition partials, rank-ordered sums -- with CPU tensors, the oracle standing
in for the kernels, and compares against the reference's single-controller
results (stencil.py:280-319, solver.py:120-189)."""

from __future__ import annotations

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dynsparse_oracle as O
from paper_2209_06478_b200 import stencil as S
from paper_2209_06478_b200.dist import HaloSchedule

SPECS = [(4, 3, 2, 2, 1, 1), (3, 4, 2, 1, 2, 1), (4, 4, 3, 1, 1, 2)]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_send_lists_equal_neighbour_plans():
    for sp in SPECS + [(4, 4, 4, 2, 2, 2), (5, 4, 3, 1, 3, 2), (3, 3, 3, 3, 3, 3)]:
        spec = S.GridSpec(*sp)
        parts = [S.generate_partition(spec, r) for r in range(spec.npartitions)]
        for p in parts:
            sched = HaloSchedule.build(spec, p)
            for q, idx, cnt, start in zip(sched.peers, sched.send_idx, sched.recv_counts,
                                          sched.recv_starts):
                theirs = {e.neighbor: e for e in parts[q].halo.exchanges}[p.rank]
                assert np.array_equal(idx, theirs.send_local_indices)
                mine = {e.neighbor: e for e in p.halo.exchanges}[q]
                assert cnt == mine.recv_ghost_slots.size
                assert start == mine.recv_ghost_slots[0]


def _exchange(sched: HaloSchedule, x_full: torch.Tensor) -> None:
    """The RankCG halo protocol on CPU tensors (pack = index_select)."""
    ops = []
    for q, idx, cnt, start in zip(sched.peers, sched.send_idx, sched.recv_counts,
                                  sched.recv_starts):
        if idx.size:
            ops.append(dist.P2POp(dist.isend, x_full[torch.from_numpy(idx)].contiguous(), q))
        if cnt:
            ops.append(dist.P2POp(dist.irecv, x_full[start:start + cnt], q))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def _gdot(local: float, world: int) -> float:
    """all-gather partials, then the reference's rank-ordered Python sum."""
    t = torch.tensor([local], dtype=torch.float64)
    out = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(out, t)
    return sum(float(v) for v in out)


def _worker(rank, world, port, sp, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        spec = S.GridSpec(*sp)
        part = S.generate_partition(spec, rank)
        sched = HaloSchedule.build(spec, part)
        n = spec.local_points
        # 1) halo exchange of random owned values vs the reference's gather
        x = torch.zeros(n + part.halo.ghost_count, dtype=torch.float64)
        x[:n] = torch.from_numpy(np.random.default_rng(100 + rank).standard_normal(n))
        _exchange(sched, x)
        oparts = O.stencil_problem(*sp)
        xs = []
        for k, p in enumerate(oparts):
            v = np.zeros(n + p.ghost_count)
            v[:n] = np.random.default_rng(100 + k).standard_normal(n)
            xs.append(v)
        O.exchange(oparts, xs)
        ok_halo = x.numpy().tobytes() == xs[rank].tobytes()
        # 2) CG with the RankCG step order: exchange, local+remote SpMV, gathered
        #    rank-ordered dots, updates -- oracle kernels on CPU
        loc, rem = O.split(oparts[rank])
        b = oparts[rank].b
        xk = np.zeros(n)
        p_full = torch.zeros(n + part.halo.ghost_count, dtype=torch.float64)
        pv = p_full.numpy()[:n]
        ap = np.zeros(n)

        def spmv_full():
            _exchange(sched, p_full)
            O.spmv(loc, pv, ap)
            O.spmv_add(rem, p_full.numpy()[n:], ap)

        spmv_full()
        r = np.zeros(n)
        O.waxpby(1.0, b, -1.0, ap, r)
        scale = math.sqrt(_gdot(O.dot(b, b), world)) or 1.0
        rr = _gdot(O.dot(r, r), world)
        hist = [math.sqrt(rr) / scale]
        O.waxpby(1.0, r, 0.0, r, pv)
        it = 0
        for it in range(1, 501):
            spmv_full()
            pap = _gdot(O.dot(pv, ap), world)
            alpha = rr / pap
            O.waxpby(1.0, xk, alpha, pv, xk)
            O.waxpby(1.0, r, -alpha, ap, r)
            rr_new = _gdot(O.dot(r, r), world)
            hist.append(math.sqrt(rr_new) / scale)
            if hist[-1] <= 1e-9:
                break
            O.waxpby(1.0, r, rr_new / rr, pv, pv)
            rr = rr_new
        ref = O.cg_dist(oparts, [O.split(p) for p in oparts], [p.b for p in oparts], tol=1e-9)
        same_hist = np.array_equal(np.asarray(hist), ref.history)
        same_x = xk.tobytes() == ref.x[rank].tobytes()
        q.put((rank, ok_halo, it == ref.iterations, same_hist, same_x))
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover - surfaced through the queue
        q.put((rank, repr(exc)))


@pytest.mark.parametrize("sp", SPECS)
def test_world2_halo_and_cg_schedule(sp):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, sp, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for res in results:
        assert len(res) == 5, res
        rank, ok_halo, same_it, same_hist, same_x = res
        assert ok_halo, f"rank {rank}: ghost slots differ from the reference exchange"
        assert same_it and same_hist and same_x, f"rank {rank}: CG differs from cg_dist"
