"""One eager PCG (MG) iteration at 104^3 after warm-up, for an ncu launch list."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_06478_b200 import hpcg  # noqa: E402
from paper_2209_06478_b200.stencil import GridSpec, generate_partition  # noqa: E402

nx = int(os.environ.get("NX", "104"))
dev = torch.device("cuda", 0)
h = hpcg.MgHierarchy.build(nx, nx, nx, device=dev)
b = generate_partition(GridSpec(nx, nx, nx), 0, hpcg.MemorySpace.DEVICE, dev).b
eng = hpcg.PcgEngine(h, b, tol=0.0, max_iters=10**6)
eng.setup()
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    eng.step(st)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("iter")
eng.step(st)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")
