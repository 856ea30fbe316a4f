"""Power-law (BASELINE config 4) conversion and plan timings, repeated (the
first call includes pool growth)."""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2209_06478_b200 as ds  # noqa: E402
from paper_2209_06478_b200 import _native, _device  # noqa: E402
dev = torch.device("cuda", 0)
rng = np.random.default_rng(2209)
n = 4_194_304
L = np.minimum(n, np.floor(6.0 * (1.0 - rng.random(n)) ** (-1 / 1.8))).astype(np.int64)
rows = np.repeat(np.arange(n, dtype=np.int64), L)
cols = rng.integers(0, n, rows.size)
vals = rng.standard_normal(rows.size)
out = {}
for rep in range(3):
    coo = ds.CooMatrix(n, n, rows, cols, vals, ds.MemorySpace.DEVICE, dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mr = ctypes.c_int32()
    _native.call("ds_coo_max_run", coo.nnz, coo.row_indices.data_ptr(), ctypes.byref(mr),
                 _device.stream(dev))
    t1 = time.perf_counter()
    csr = ds.convert(coo, ds.FormatId.CSR)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out[f"rep{rep}"] = {"max_run_ms": round((t1 - t0) * 1e3, 2), "max_run": mr.value,
                        "convert_ms": round((t2 - t1) * 1e3, 2)}
print(json.dumps(out))
