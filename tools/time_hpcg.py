"""Time the device SymGS sweep, V-cycle and one PCG solve (CUDA events)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_06478_b200 import hpcg  # noqa: E402
from paper_2209_06478_b200.stencil import GridSpec, generate_partition  # noqa: E402

nx = int(os.environ.get("NX", "104"))
dev = torch.device("cuda", 0)
t0 = time.time()
h = hpcg.MgHierarchy.build(nx, nx, nx, device=dev, layout=os.environ.get("LAYOUT", "ell"))
torch.cuda.synchronize()
print("build", [L.nrows for L in h.levels], f"{time.time() - t0:.2f}s")
n = h.levels[0].nrows
nnz = h.levels[0].a.nnz
r = torch.randn(n, dtype=torch.float64, device=dev)
x = torch.zeros(n, dtype=torch.float64, device=dev)


def timeit(fn, reps=50):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


us = timeit(lambda: h.symgs(0, r, x))
byts = 15 / 8 * (n * (26 * 12 + 8 + 4 + 4) + n * 8 * 3)
print(f"symgs {us:.1f} us  ({byts / us / 1e3:.0f} GB/s algorithmic, 2 sweeps)")
us = timeit(lambda: h.vcycle(r, x))
print(f"vcycle {us:.1f} us")
b = generate_partition(GridSpec(nx, nx, nx), 0, hpcg.MemorySpace.DEVICE, dev).b
torch.cuda.synchronize()
t0 = time.time()
res = hpcg.pcg(h, b, tol=1e-9, max_iters=50)
torch.cuda.synchronize()
dt = time.time() - t0
print(f"pcg iters {res.iterations} conv {res.converged} {dt * 1e3:.1f} ms "
      f"({dt / max(res.iterations, 1) * 1e6:.0f} us/iter) final {res.residual_history[-1]:.3e}")
eng = hpcg.PcgEngine(h, b, tol=0.0, max_iters=10**6)
eng.setup()
eng._capture(1)
us = timeit(eng.graph.replay, reps=20)
print(f"pcg iteration (graph) {us:.1f} us")
eng2 = hpcg.PcgEngine(h, b, tol=0.0, max_iters=10**6)
eng2.setup()
st = torch.cuda.current_stream().cuda_stream
us = timeit(lambda: eng2.step(st), reps=20)
print(f"pcg iteration (eager) {us:.1f} us")
