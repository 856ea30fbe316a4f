"""Device timeline (torch.profiler / CUPTI) of single conversions at NX^3
after warm-up: every kernel / memcpy / memset with its start offset and
duration, and the idle gaps between them (host syncs, allocations)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402
import paper_2209_06478_b200 as ds  # noqa: E402
nx = int(os.environ.get("NX", "192"))
dev = torch.device("cuda", 0)
part = ds.generate_partition(ds.GridSpec(nx, nx, nx), 0, space=ds.MemorySpace.DEVICE, device=dev)
mats = {"csr": part.a_full}
mats["dia"] = ds.convert(part.a_full, ds.FormatId.DIA)
mats["coo"] = ds.convert(part.a_full, ds.FormatId.COO)
pairs = [p.split("-") for p in os.environ.get("PAIRS", "csr-dia dia-csr csr-coo coo-csr").split()]
for s, d in pairs:
    for _ in range(2):
        ds.convert(mats[s], ds.FormatId[d.upper()])
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        ds.convert(mats[s], ds.FormatId[d.upper()])
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    if not ev:
        print(s, d, "no device events")
        continue
    t0 = ev[0].time_range.start
    end = t0
    busy = 0.0
    print(f"== {s}->{d}")
    for e in ev:
        st, du = e.time_range.start, e.time_range.end - e.time_range.start
        gap = st - end
        busy += du
        print(f"  +{st - t0:8.1f} us  gap {gap:7.1f}  {du:8.1f} us  {e.name[:70]}")
        end = max(end, e.time_range.end)
    print(f"  device span {end - t0:.1f} us, busy {busy:.1f} us")
