import cProfile, pstats, os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2209_06478_b200 as ds
dev = torch.device("cuda", 0)
spec = ds.GridSpec(104, 104, 104)
part = ds.generate_partition(spec, 0, space=ds.MemorySpace.DEVICE, device=dev)
split = ds.split_local_remote(ds.PartitionedProblem(spec, [part]), 0)
ds.convert_inplace(split.local, ds.FormatId.DIA)
op = ds.DistributedOperator(ds.PartitionedProblem(spec, [part]), [split])
b_host = ds.DenseVector(part.b.data.cpu().numpy())
for _ in range(3):
    ds.cg(ds.SERIAL, op, [b_host])
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    ds.cg(ds.SERIAL, op, [b_host])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
