"""One rank of a multi-process CG run (launched by torch.distributed.run from
tests/test_gpu_multirank.py or by hand).

Every rank drives the GPU ``LOCAL_RANK % device_count`` -- on a one-GPU box
all ranks share cuda:0 and the peer transport's IPC mappings alias the same
HBM; on an 8-GPU node each rank has its own device.  torch.distributed
(gloo) only bootstraps.  Each rank writes rank<r>.npz (iterations, history,
owned x, the morpheus / ghost / multi plans) into --out.
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, nargs=3, required=True)
    ap.add_argument("--procs", type=int, nargs=3, required=True)
    ap.add_argument("--local-format", default="dia")
    ap.add_argument("--transport", default="peer")
    ap.add_argument("--tol", type=float, default=1e-9)
    ap.add_argument("--max-iters", type=int, default=500)
    ap.add_argument("--graph-steps", type=int, default=1)
    ap.add_argument("--tune", action="store_true", help="also run the per-rank tuner")
    ap.add_argument("--out", required=True)
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2209_06478_b200 as ds
    from paper_2209_06478_b200 import dist as D

    rank = int(os.environ["RANK"])
    if os.environ.get("DS_TEST_NCCL_FAKE_HOSTS") == "1":
        # several NCCL ranks on ONE GPU: NCCL refuses two ranks of a
        # communicator on one device of one host, so each rank claims its own
        # host id and the ranks talk through NCCL's socket transport (loopback)
        os.environ["NCCL_HOSTID"] = f"ds-test-host-{rank}"
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    spec = ds.GridSpec(*args.grid, *args.procs)
    assert spec.npartitions == world, (spec.npartitions, world)
    part = ds.generate_partition(spec, rank, space=ds.MemorySpace.DEVICE, device=dev)
    split = ds.split_local_remote(ds.PartitionedProblem(spec, [part]), 0)
    plans = {}
    if args.tune:
        prof = D.profile_rank(part, split, reps=3)
        for mode in ("multi", "morpheus", "ghost"):
            lf, rf = D.select_rank_plan(prof["entries"], mode, world)
            plans[mode] = (int(lf), int(rf))
        # amortised selection must also be consistent across ranks
        lf, rf = D.select_rank_plan(prof["entries"], "morpheus", world, prof["convert_s"], 50)
        plans["morpheus_amortised"] = (int(lf), int(rf))
    ds.convert_inplace(split.local, ds.FormatId[args.local_format.upper()])
    eng = D.RankCG(spec, part, split, dev, args.tol, args.max_iters, transport=args.transport)
    try:
        if args.graph_steps > 1:
            eng.capture_step(args.graph_steps)
        x, it, hist, conv = eng.solve()
        xs = x.data.cpu().numpy()
    finally:
        eng.close()
    np.savez(os.path.join(args.out, f"rank{rank}.npz"), iterations=it, history=hist, x=xs,
             converged=conv, plans=np.array([plans.get(m, (-1, -1)) for m in
                                             ("multi", "morpheus", "ghost",
                                              "morpheus_amortised")]))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
