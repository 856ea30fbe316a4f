"""ncu --csv launch list (one row per metric) -> one row per launch:
id,kernel,time_ns,dram_read_bytes,dram_write_bytes.  Usage:
python tools/compact_launches.py launches.csv > out.csv"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
h = rows[0]
ii, ki, mi, ui, vi = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Unit",
                                            "Metric Value"))
scale = {"ns": 1, "us": 1e3, "usecond": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = OrderedDict()
for r in rows[1:]:
    d = out.setdefault(r[ii], {"kernel": r[ki].split("(")[0][:80]})
    d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
w = csv.writer(sys.stdout)
w.writerow(["id", "kernel", "time_ns", "dram_read_bytes", "dram_write_bytes"])
for i, d in out.items():
    w.writerow([i, d["kernel"], round(d.get("gpu__time_duration.sum", 0)),
                round(d.get("dram__bytes_read.sum", 0)), round(d.get("dram__bytes_write.sum", 0))])
