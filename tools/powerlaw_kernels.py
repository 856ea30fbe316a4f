"""Power-law (BASELINE config 4) SpMV + conversion timings, and a short mode
for ncu (PROFILE=1: each SpMV launched twice after one warm-up).

    python tools/powerlaw_kernels.py            # timings (JSON)
    PROFILE=1 ncu ... python tools/powerlaw_kernels.py
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2209_06478_b200 as ds  # noqa: E402
from paper_2209_06478_b200.kernels import prepared_spmv  # noqa: E402

dev = torch.device("cuda", 0)
prof = os.environ.get("PROFILE") == "1"
fmts = os.environ.get("FMTS", "csr,coo").split(",")
rng = np.random.default_rng(2209)
n = 4_194_304
L = np.minimum(n, np.floor(6.0 * (1.0 - rng.random(n)) ** (-1 / 1.8))).astype(np.int64)
rows = np.repeat(np.arange(n, dtype=np.int64), L)
cols = rng.integers(0, n, rows.size)
vals = rng.standard_normal(rows.size)
out = {}
conv = []
for rep in range(1 if prof else 3):
    coo = ds.CooMatrix(n, n, rows, cols, vals, ds.MemorySpace.DEVICE, dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    csr = ds.convert(coo, ds.FormatId.CSR)
    torch.cuda.synchronize()
    conv.append(round((time.perf_counter() - t0) * 1e3, 3))
    del coo
out["coo_to_csr_ms"] = conv
ccoo = ds.convert(csr, ds.FormatId.COO)
x = ds.DenseVector(torch.from_numpy(np.random.default_rng(1).standard_normal(n)).to(dev))
y = ds.DenseVector.zeros(n, ds.MemorySpace.DEVICE, dev)
nnz = csr.nnz
for name in fmts:
    m = csr if name == "csr" else ccoo
    launch = prepared_spmv(m, x, y, 0)
    launch()
    if prof:
        launch()
        launch()
        torch.cuda.synchronize()
        continue
    for _ in range(5):
        launch()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(10)]
    st = torch.cuda.current_stream()
    for a, b in ev:
        a.record(st)
        for _ in range(5):
            launch()
        b.record(st)
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) / 5 for a, b in ev)
    bytes_ = (12 * nnz + 4 * (n + 1) + 16 * n) if name == "csr" else (16 * nnz + 16 * n)
    out[name] = {"us": round(ms * 1e3, 1), "gbs": round(bytes_ / ms / 1e6, 1)}
print(json.dumps(out))
