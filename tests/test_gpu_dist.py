"""GPU: the one-partition-per-process engine (dist.RankCG: NCCL halo +
all-gather dots, CUDA-graph step) at world size 1 -- the only size a single
B200 allows -- against the oracle's CG."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2209_06478_b200 as ds  # noqa: E402
from paper_2209_06478_b200 import dist as D  # noqa: E402
from oracle import dynsparse_oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def pg():
    import torch.distributed as dist
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("fmt", ["csr", "dia", "coo"])
def test_rank_cg_world1_matches_oracle(pg, fmt):
    dev = torch.device("cuda", 0)
    spec = ds.GridSpec(12, 10, 8)
    part = ds.generate_partition(spec, 0, space=ds.MemorySpace.DEVICE, device=dev)
    split = ds.split_local_remote(ds.PartitionedProblem(spec, [part]), 0)
    ds.convert_inplace(split.local, ds.FormatId[fmt.upper()])
    x, it, hist, conv = D.rank_cg(spec, part, split, tol=1e-9, max_iters=500, device=dev,
                                  transport="nccl")
    op = O.stencil_partition(12, 10, 8)
    loc, rem = O.split(op)
    ref = O.cg_dist([op], [(loc, rem)], [op.b], tol=1e-9)
    assert conv and abs(it - ref.iterations) <= 1
    k = min(it, ref.iterations) + 1
    assert np.all(np.abs(hist[:k] - ref.history[:k]) <= 1e-8 * ref.history[:k] + 1e-14)
    assert np.max(np.abs(x.data.cpu().numpy() - ref.x[0])) < 1e-8


@pytest.mark.parametrize("fmt", ["dia", "csr"])
def test_rank_cg_world1_peer_transport(pg, fmt):
    """World size 1 through the peer transport (self-exchange of the dots)."""
    dev = torch.device("cuda", 0)
    spec = ds.GridSpec(10, 9, 8)
    part = ds.generate_partition(spec, 0, space=ds.MemorySpace.DEVICE, device=dev)
    split = ds.split_local_remote(ds.PartitionedProblem(spec, [part]), 0)
    ds.convert_inplace(split.local, ds.FormatId[fmt.upper()])
    x, it, hist, conv = D.rank_cg(spec, part, split, tol=1e-9, device=dev, transport="peer")
    op = O.stencil_partition(10, 9, 8)
    ref = O.cg_dist([op], [O.split(op)], [op.b], tol=1e-9)
    assert conv and abs(it - ref.iterations) <= 1
    k = min(it, ref.iterations) + 1
    assert np.all(np.abs(hist[:k] - ref.history[:k]) <= 1e-8 * ref.history[:k] + 1e-14)


def test_nccl_halo_exchange_self_peer_guard(pg):
    """ds_halo_exchange at world size 1 with rank 0 as its own neighbour: the
    send list lands in the rank's own ghost slots in one NCCL group.  While
    s->done == 0 (and r.r holds a non-integer, the value the old guard
    mistook for the flag) the ghosts refresh on every exchange; once done is
    set the packs are skipped and the ghosts keep their last values."""
    import ctypes

    from paper_2209_06478_b200 import _native
    lib = _native.load()
    dev = torch.device("cuda", 0)
    comm, _, _ = D.init_comm(dev)
    try:
        n, g = 64, 12
        idx = torch.arange(5, 5 + g, dtype=torch.int32, device=dev) * 3 % n
        x = torch.zeros(n + g, dtype=torch.float64, device=dev)
        sbuf = torch.zeros(g, dtype=torch.float64, device=dev)
        scal = torch.zeros(_native.CG_SCALARS_BYTES // 8, dtype=torch.float64, device=dev)
        arr = lambda ty, v: (ty * len(v))(*v)  # noqa: E731
        args = (1, arr(ctypes.c_int32, [0]), arr(ctypes.c_int64, [g]),
                arr(ctypes.c_void_p, [idx.data_ptr()]), arr(ctypes.c_void_p, [sbuf.data_ptr()]),
                arr(ctypes.c_int64, [g]), arr(ctypes.c_int64, [n]))
        st = torch.cuda.current_stream(dev).cuda_stream
        for it in range(4):
            x[:n] = torch.arange(n, dtype=torch.float64, device=dev) * (it + 1.5)
            scal[0] = 2.0 ** 0.5 * (it + 1)      # rr: non-integer, low word nonzero
            _native.check(lib.ds_halo_exchange(*args, x.data_ptr(), scal.data_ptr(), comm, st))
            torch.cuda.synchronize(dev)
            assert torch.equal(x[n:], x[:n][idx.long()]), f"ghosts stale at exchange {it}"
        frozen = x[n:].clone()
        sc = _native.DsCgScalars.from_buffer_copy(scal.cpu().numpy().tobytes())
        sc.done = 1
        scal.copy_(torch.frombuffer(bytearray(bytes(sc)), dtype=torch.float64).to(dev))
        x[:n] = -7.0
        _native.check(lib.ds_halo_exchange(*args, x.data_ptr(), scal.data_ptr(), comm, st))
        torch.cuda.synchronize(dev)
        assert torch.equal(x[n:], frozen), "ghosts changed after done was set"
    finally:
        _native.check(lib.ds_nccl_comm_destroy(comm))
