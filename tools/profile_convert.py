"""One CSR->DIA and one DIA->CSR conversion at NX^3 after warm-up (ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2209_06478_b200 as ds  # noqa: E402
nx = int(os.environ.get("NX", "192"))
dev = torch.device("cuda", 0)
part = ds.generate_partition(ds.GridSpec(nx, nx, nx), 0, space=ds.MemorySpace.DEVICE, device=dev)
a = part.a_full
for _ in range(2):
    d = ds.convert(a, ds.FormatId.DIA)
    c = ds.convert(d, ds.FormatId.CSR)
    o = ds.convert(a, ds.FormatId.COO)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("measured")
d = ds.convert(a, ds.FormatId.DIA)
c = ds.convert(d, ds.FormatId.CSR)
o = ds.convert(a, ds.FormatId.COO)
torch.cuda.synchronize()
print("done")
