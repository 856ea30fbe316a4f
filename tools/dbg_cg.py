import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2209_06478_b200 as ds
from oracle import dynsparse_oracle as O
dev = torch.device("cuda", 0)
for sp in [(3,3,3,1,1,1),(4,3,2,2,1,1),(4,4,4,2,2,2)]:
    spec = ds.GridSpec(*sp)
    prob = ds.generate_problem(spec, space=ds.MemorySpace.DEVICE, device=dev)
    splits = [ds.split_local_remote(prob, k) for k in range(prob.npartitions)]
    res = ds.cg(ds.SERIAL, ds.DistributedOperator(prob, splits), [p.b for p in prob.partitions], tol=1e-9, max_iters=500, use_graph=False)
    parts = O.stencil_problem(*sp); osp = [O.split(p) for p in parts]
    ref = O.cg_dist(parts, osp, [p.b for p in parts], tol=1e-9)
    print(sp, "dist", res.iterations, ref.iterations, res.residual_history[:4], ref.history[:4])
    if spec.npartitions == 1:
        r2 = ds.cg(ds.SERIAL, prob.partitions[0].a_full, prob.partitions[0].b, tol=1e-9, use_graph=False)
        print("   single", r2.iterations, r2.residual_history[:4])
        a = prob.partitions[0].a_full
        x = ds.DenseVector.ones(a.ncols, ds.MemorySpace.DEVICE, dev); y = ds.DenseVector.zeros(a.nrows, ds.MemorySpace.DEVICE, dev)
        ds.spmv(ds.SERIAL, a, x, y); print("   A*1 == b:", torch.equal(y.data, prob.partitions[0].b.data))
        ds.dot(ds.SERIAL, y, y)
