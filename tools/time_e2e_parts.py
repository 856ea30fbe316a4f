"""Where the e2e cg() time goes (104^3, host b -> host x): per-stage wall
times of the cached-engine path (reload / device solve / history / x out)."""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2209_06478_b200 as ds  # noqa: E402
from paper_2209_06478_b200 import solver as S  # noqa: E402

dev = torch.device("cuda", 0)
spec = ds.GridSpec(104, 104, 104)
part = ds.generate_partition(spec, 0, space=ds.MemorySpace.DEVICE, device=dev)
split = ds.split_local_remote(ds.PartitionedProblem(spec, [part]), 0)
ds.convert_inplace(split.local, ds.FormatId.DIA)
op = ds.DistributedOperator(ds.PartitionedProblem(spec, [part]), [split])
b_host = ds.DenseVector(part.b.data.cpu().numpy())
for _ in range(3):
    ds.cg(ds.SERIAL, op, [b_host])
eng = op.__dict__["_cg_engine"][1]
T = {k: [] for k in ("total", "reload", "run", "finish", "xout")}
for _ in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S._reload(eng, [b_host], None)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    sc = eng.run()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    it, hist, conv = S._finish(eng, sc)
    t3 = time.perf_counter()
    o = S._pinned(eng, "x0", eng.parts[0].n)
    o.copy_(eng.parts[0].x, non_blocking=True)
    torch.cuda.synchronize()
    x = torch.empty_like(o).copy_(o).numpy()
    t4 = time.perf_counter()
    for k, v in zip(T, (t4 - t0, t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
        T[k].append(v * 1e3)
    tt = time.perf_counter()
    ds.cg(ds.SERIAL, op, [b_host])
    T.setdefault("cg_call", []).append((time.perf_counter() - tt) * 1e3)
print(json.dumps({k: round(statistics.median(v), 3) for k, v in T.items()} | {"iterations": it,
      "torch_threads": torch.get_num_threads()}))
