"""Per-level SymGS time (graph of 20 calls, CUDA events) for the MG hierarchy."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_06478_b200 import hpcg  # noqa: E402

nx = int(os.environ.get("NX", "104"))
dev = torch.device("cuda", 0)
h = hpcg.MgHierarchy.build(nx, nx, nx, device=dev)
out = []
for lev, L in enumerate(h.levels):
    n = L.nrows
    r = torch.randn(n, dtype=torch.float64, device=dev)
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    side = torch.cuda.Stream()
    for _ in range(2):
        h.symgs(lev, r, x)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(20):
            h.symgs(lev, r, x, st=side.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    out.append((lev, n, round(a.elapsed_time(b) * 1e3 / 20, 1)))
print(os.environ.get("DS_SYMGS_CLUSTER_ROWS", "default"), out)
