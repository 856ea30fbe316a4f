"""HPCG PCG-MG at 104^3: a graph of 20 full iterations vs 20 V-cycles alone vs
20 x (SpMV + dots + axpys) alone -- where the iteration's time goes."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2209_06478_b200 import hpcg  # noqa: E402
from paper_2209_06478_b200.stencil import GridSpec, generate_partition  # noqa: E402

nx = int(os.environ.get("NX", "104"))
dev = torch.device("cuda", 0)
h = hpcg.MgHierarchy.build(nx, nx, nx, device=dev)
b = generate_partition(GridSpec(nx, nx, nx), 0, hpcg.MemorySpace.DEVICE, dev).b
eng = hpcg.PcgEngine(h, b, tol=0.0, max_iters=10**6)
eng.setup()
side = torch.cuda.Stream()
sp = side.cuda_stream
orig_vcycle = h.vcycle


def graph_of(body):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(20):
            body()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(e) * 1e3 / 20)
    return round(statistics.median(ts), 1)


out = {"iteration_us": graph_of(lambda: eng.step(sp)),
       "vcycle_us": graph_of(lambda: h.vcycle(eng.r, eng.z, 0, sp))}
h.vcycle = lambda r, z, lev=0, st=None: None   # the rest of the iteration only
out["rest_us"] = graph_of(lambda: eng.step(sp))
h.vcycle = orig_vcycle
print(json.dumps(out))
