"""One conversion (env SRC, DST, NX) for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2209_06478_b200 as ds  # noqa: E402
nx = int(os.environ.get("NX", "104"))
dev = torch.device("cuda", 0)
part = ds.generate_partition(ds.GridSpec(nx, nx, nx), 0, space=ds.MemorySpace.DEVICE, device=dev)
m = ds.convert(part.a_full, ds.FormatId[os.environ.get("SRC", "csr").upper()])
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("convert")
ds.convert(m, ds.FormatId[os.environ.get("DST", "dia").upper()])
torch.cuda.synchronize()
