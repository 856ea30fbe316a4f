"""Time y = A x at 104^3 for one format (env FMT) -- for tile-shape sweeps
(DS_DIA_T / DS_DIA_S / DS_DIA_CTAS ...).  Prints one JSON line."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2209_06478_b200 as ds  # noqa: E402

fmt = os.environ.get("FMT", "dia")
nx = int(os.environ.get("NX", "104"))
dev = torch.device("cuda", 0)
if os.environ.get("POWERLAW"):
    rng = np.random.default_rng(2209)
    n = 4_194_304
    L = np.minimum(n, np.floor(6.0 * (1.0 - rng.random(n)) ** (-1 / 1.8))).astype(np.int64)
    if os.environ.get("POWERLAW_CAP"):   # experiment: cap row lengths
        L = np.minimum(L, int(os.environ["POWERLAW_CAP"]))
    rows = np.repeat(np.arange(n, dtype=np.int64), L)
    a_csr = ds.convert(ds.CooMatrix(n, n, rows, rng.integers(0, n, rows.size),
                                    rng.standard_normal(rows.size), ds.MemorySpace.DEVICE, dev),
                       ds.FormatId.CSR)

    class _P:  # stand-in for a partition
        a_full = a_csr
    part = _P()
else:
    part = ds.generate_partition(ds.GridSpec(nx, nx, nx), 0, space=ds.MemorySpace.DEVICE, device=dev)
n = part.a_full.nrows
x = ds.DenseVector(torch.from_numpy(np.random.default_rng(0).standard_normal(n)).to(dev))
y = ds.DenseVector.zeros(n, ds.MemorySpace.DEVICE, dev)
m = ds.convert(part.a_full, ds.FormatId[fmt.upper()])
ref = ds.DenseVector.zeros(n, ds.MemorySpace.DEVICE, dev)
ds.spmv(ds.SERIAL, ds.convert(part.a_full, ds.FormatId.CSR), x, ref)
from paper_2209_06478_b200.kernels import prepared_spmv  # noqa: E402
launch = prepared_spmv(m, x, y, 0)
for _ in range(20):
    launch()
st = torch.cuda.current_stream()
# batches of back-to-back launches (the device never waits for Python)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
for a, b in ev:
    a.record(st)
    for _ in range(40):
        launch()
    b.record(st)
torch.cuda.synchronize()
ms = statistics.median(a.elapsed_time(b) / 40 for a, b in ev)
nnz = part.a_full.nnz
byts = {"dia": 8 * getattr(m, "ndiags", 27) * n + 16 * n, "csr": 12 * nnz + 4 * (n + 1) + 16 * n,
        "coo": 16 * nnz + 16 * n}[fmt]
err = float(torch.linalg.norm(y.data - ref.data) / torch.linalg.norm(ref.data))
print(json.dumps({"fmt": fmt, "env": {k: v for k, v in os.environ.items() if k.startswith("DS_")},
                  "us": round(ms * 1e3, 2), "GBs": round(byts / ms / 1e6, 1),
                  "GFs": round(2 * nnz / ms / 1e6, 1), "relerr_vs_csr": err}))
