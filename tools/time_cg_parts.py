"""Graph-captured CG step variants at 104^3 (timing experiments only; the
partial variants compute garbage): full step vs without the direction kernel
vs SpMV alone.  Each graph holds 20 steps, replayed 50 times."""
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
ds.convert_inplace(split.local, ds.FormatId.DIA)
eng, _ = S.build_engine(S.DistributedOperator(prob, [split]), [part.b], None, 1e-300, 10**9)
side = torch.cuda.Stream()
sp = side.cuda_stream
eng.setup(sp)
lib, s, hist, ws = eng.lib, eng._p(eng.scal), eng._p(eng.hist), eng._p(eng.ws)
pt = eng.parts[0]
spmv = lambda: lib.ds_cg_spmv_dot(ctypes.byref(pt.d_local), eng._p(pt.p_full), eng._p(pt.ap),  # noqa
                                  pt.local_mode, eng._p(pt.p), eng._dot(2, 0), S.DEFERRED, s,
                                  hist, None, 0, ws, sp)
upd = lambda: lib.ds_cg_update_deferred(pt.n, eng._p(pt.x), eng._p(pt.r), eng._p(pt.p),  # noqa
                                        eng._p(pt.ap), s, ws, sp)
dirn = lambda: lib.ds_cg_direction_deferred(pt.n, eng._p(pt.r), eng._p(pt.p), s, hist, ws, sp)  # noqa
fused = lambda: lib.ds_cg_update_direction_deferred(pt.n, eng._p(pt.x), eng._p(pt.r),  # noqa
                                                    eng._p(pt.p), eng._p(pt.ap), s, hist, ws, sp)
variants = {"full": (spmv, upd, dirn), "fused": (spmv, fused), "no_direction": (spmv, upd), "spmv_only": (spmv,),
            "spmv_direction": (spmv, dirn), "tail_only": (fused,), "update_only": (upd,),
            "direction_only": (dirn,)}
cudart = ctypes.CDLL("libcudart.so.12") if False else None
try:
    from cuda.bindings import runtime as rt
    attrs = {}
    for nm in ("cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize",
               "cudaDevAttrL2CacheSize"):
        err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, nm), 0)
        attrs[nm] = v
    print(json.dumps(attrs), file=sys.stderr)
except Exception as e:  # noqa: BLE001
    print("attrs:", e, file=sys.stderr)
out = {}
if os.environ.get("PERSIST") == "1":   # the bench's persisting-L2 window over the CG vectors
    vb = eng.parts[0].vec_block
    print("persist rc", lib.ds_l2_persist(vb.data_ptr(), vb.numel() * 8, sp), file=sys.stderr)
for name, fns in variants.items():
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(20):
            for f in fns:
                f()
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    ts = []
    for _ in range(50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / 20)
    out[name] = round(statistics.median(ts), 2)
print(json.dumps({"persist": os.environ.get("PERSIST") == "1", "us_per_step": out}))
