"""Where the e2e cg() time goes (104^3, host b -> host x): per-stage wall
times of the cached-engine path (reload / setup / device loop / history /
x out), CUDA-synchronised between stages."""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2209_06478_b200 as ds  # noqa: E402
from paper_2209_06478_b200 import _native, _device  # noqa: E402
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
T = {}
def mark(k, t0):
    torch.cuda.synchronize()
    t = time.perf_counter()
    T.setdefault(k, []).append((t - t0) * 1e3)
    return t
for _ in range(10):
    torch.cuda.synchronize()
    t = t0 = time.perf_counter()
    S._reload(eng, [b_host], None)
    t = mark("reload", t)
    st = _device.stream(dev)
    eng.setup(st)
    t = mark("setup", t)
    eng._persist_on(st)   # as CgEngine.run does before a cached-graph launch
    _native.check(eng.lib.ds_graph_exec_launch(eng._while[1], st))
    t = mark("while_loop", t)
    eng.release_l2(st)
    sc = eng.scalars()
    t = mark("scalars", t)
    it, hist, conv = S._finish(eng, sc)
    t = mark("history", t)
    outs = [S._pinned_result(eng, 0, eng.parts[0].n)]
    outs[0][0].copy_(eng.parts[0].x, non_blocking=True)
    x = np.ctypeslib.as_array(outs[0][1])
    t = mark("x_out", t)
    T.setdefault("total", []).append((t - t0) * 1e3)
    del x
    tt = time.perf_counter()
    r = ds.cg(ds.SERIAL, op, [b_host])
    T.setdefault("cg_call", []).append((time.perf_counter() - tt) * 1e3)
    del r
print(json.dumps({k: round(statistics.median(v), 3) for k, v in T.items()} | {"iterations": it}))
