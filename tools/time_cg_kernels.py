"""Per-kernel CUDA-event times inside eager single-partition CG steps at
104^3 (DIA local): spmv+p.Ap | update | direction, plus the graph step."""
import ctypes, json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2209_06478_b200 as ds  # noqa: E402
from paper_2209_06478_b200 import solver as S  # noqa: E402

nx = int(os.environ.get("NX", "104"))
dev = torch.device("cuda", 0)
spec = ds.GridSpec(nx, nx, nx)
part = ds.generate_partition(spec, 0, space=ds.MemorySpace.DEVICE, device=dev)
prob = ds.PartitionedProblem(spec, [part])
split = ds.split_local_remote(prob, 0)
ds.convert_inplace(split.local, ds.FormatId[os.environ.get("FMT", "dia").upper()])
eng, _ = S.build_engine(S.DistributedOperator(prob, [split]), [part.b], None, 1e-300, 100000)
st = torch.cuda.current_stream()
sp = st.cuda_stream
eng.setup(sp)
lib, s, hist, ws = eng.lib, eng._p(eng.scal), eng._p(eng.hist), eng._p(eng.ws)
pt = eng.parts[0]
calls = {
    "spmv": lambda sp: lib.ds_cg_spmv_dot(ctypes.byref(pt.d_local), eng._p(pt.p_full),
                                          eng._p(pt.ap), pt.local_mode, eng._p(pt.p),
                                          eng._dot(2, 0), S.DEFERRED, s, hist, None, 0, ws, sp),
    "update": lambda sp: lib.ds_cg_update_deferred(pt.n, eng._p(pt.x), eng._p(pt.r),
                                                   eng._p(pt.p), eng._p(pt.ap), s, ws, sp),
    "direction": lambda sp: lib.ds_cg_direction_deferred(pt.n, eng._p(pt.r), eng._p(pt.p), s,
                                                         hist, ws, sp),
}
# one CUDA graph per kernel (eager ctypes launches are CPU bound), replayed
# back to back with events between them
side = torch.cuda.Stream()
graphs = {}
for k, fn in calls.items():
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        fn(side.cuda_stream)
    graphs[k] = g
torch.cuda.synchronize()
names = list(calls)
ts = {k: [] for k in names + ["step"]}
for it in range(220):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(st)
    for j, k in enumerate(names):
        graphs[k].replay()
        ev[j + 1].record(st)
    if it >= 20:
        torch.cuda.synchronize()
        for j, k in enumerate(names):
            ts[k].append(ev[j].elapsed_time(ev[j + 1]) * 1e3)
        ts["step"].append(ev[0].elapsed_time(ev[3]) * 1e3)
print(json.dumps({"fmt": os.environ.get("FMT", "dia"),
                  **{k: round(statistics.median(v), 2) for k, v in ts.items()}}))
