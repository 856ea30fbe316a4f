"""Wall time of ds.cg() from a host b to a host x at 104^3 for several
iteration counts (intercept = fixed per-call overhead), with a cProfile of
one 50-iteration call."""
import cProfile
import os
import pstats
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2209_06478_b200 as ds  # noqa: E402

dev = torch.device("cuda", 0)
spec = ds.GridSpec(104, 104, 104)
part = ds.generate_partition(spec, 0, space=ds.MemorySpace.DEVICE, device=dev)
split = ds.split_local_remote(ds.PartitionedProblem(spec, [part]), 0)
ds.convert_inplace(split.local, ds.FormatId.DIA)
op = ds.DistributedOperator(ds.PartitionedProblem(spec, [part]), [split])
b_host = ds.DenseVector(part.b.data.cpu().numpy())
for iters in (1, 10, 50, 200):
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ds.cg(ds.SERIAL, op, [b_host], tol=1e-300, max_iters=iters)
        ts.append(time.perf_counter() - t0)
    print(iters, round(statistics.median(ts[1:]) * 1e3, 3), "ms")
ts = []
for _ in range(7):   # the reference's defaults (tol 1e-9): converges
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = ds.cg(ds.SERIAL, op, [b_host])
    ts.append(time.perf_counter() - t0)
print("default tol:", res.iterations, "iterations", round(statistics.median(ts[1:]) * 1e3, 3), "ms")
if os.environ.get("NO_PROFILE"):
    sys.exit(0)
pr = cProfile.Profile()
pr.enable()
ds.cg(ds.SERIAL, op, [b_host], tol=1e-300, max_iters=50)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
