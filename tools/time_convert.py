"""Wall time (CUDA-synchronised) of every format conversion at 104^3 (or NX)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2209_06478_b200 as ds  # noqa: E402
nx = int(os.environ.get("NX", "104"))
dev = torch.device("cuda", 0)
part = ds.generate_partition(ds.GridSpec(nx, nx, nx), 0, space=ds.MemorySpace.DEVICE, device=dev)
mats = {"csr": part.a_full}
out = {}
for src in ("csr", "coo", "dia"):
    for dst in ("csr", "coo", "dia"):
        if src not in mats:
            mats[src] = ds.convert(part.a_full, ds.FormatId[src.upper()])
        m = mats[src]
        ds.convert(m, ds.FormatId[dst.upper()])   # warm
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            ds.convert(m, ds.FormatId[dst.upper()])
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        out[f"{src}->{dst}"] = round(min(ts) * 1e3, 3)
import bench  # noqa: E402
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
fl = bench.convert_floor(out, part.a_full.nrows, part.a_full.nnz, mats["dia"].ndiags, peak)
print(json.dumps({"nx": nx, "convert_ms": out,
                  "frac_of_byte_floor": {k: v["frac"] for k, v in fl.items()}}))
