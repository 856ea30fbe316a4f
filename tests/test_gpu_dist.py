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
    x, it, hist, conv = D.rank_cg(spec, part, split, tol=1e-9, max_iters=500, device=dev)
    op = O.stencil_partition(12, 10, 8)
    loc, rem = O.split(op)
    ref = O.cg_dist([op], [(loc, rem)], [op.b], tol=1e-9)
    assert conv and abs(it - ref.iterations) <= 1
    k = min(it, ref.iterations) + 1
    assert np.all(np.abs(hist[:k] - ref.history[:k]) <= 1e-8 * ref.history[:k] + 1e-14)
    assert np.max(np.abs(x.data.cpu().numpy() - ref.x[0])) < 1e-8
