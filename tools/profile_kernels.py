"""Small driver for ncu: 104^3 stencil, each SpMV format a few times, then a
few eager CG steps (fused DIA SpMV + update + direction).  Used by
tools/ncu.sh; never a source of bench numbers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2209_06478_b200 as ds  # noqa: E402
from paper_2209_06478_b200 import solver as S  # noqa: E402

reps = int(os.environ.get("REPS", "3"))
dev = torch.device("cuda", 0)
spec = ds.GridSpec(104, 104, 104)
part = ds.generate_partition(spec, 0, space=ds.MemorySpace.DEVICE, device=dev)
n = part.a_full.nrows
x = ds.DenseVector(torch.from_numpy(np.random.default_rng(0).standard_normal(n)).to(dev))
y = ds.DenseVector.zeros(n, ds.MemorySpace.DEVICE, dev)
mats = {f: ds.convert(part.a_full, f) for f in (ds.FormatId.DIA, ds.FormatId.CSR, ds.FormatId.COO)}
torch.cuda.synchronize()
for f, m in mats.items():
    for _ in range(reps):
        ds.spmv(ds.SERIAL, m, x, y)
torch.cuda.synchronize()
prob = ds.PartitionedProblem(spec, [part])
split = ds.split_local_remote(prob, 0)
ds.convert_inplace(split.local, ds.FormatId.DIA)
eng, _ = S.build_engine(S.DistributedOperator(prob, [split]), [part.b], None, 1e-300, 100)
st = torch.cuda.current_stream().cuda_stream
eng.setup(st)
for _ in range(reps):
    eng.step(st)
torch.cuda.synchronize()
print("profile driver done")
