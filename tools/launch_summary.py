"""Summarise an ncu --csv launch list: total time per kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot, cnt = defaultdict(float), defaultdict(int)
launches = [r for r in rows[1:] if r[mi] == "gpu__time_duration.sum"][skip:]
for r in launches:
    name = r[ki].split("(")[0].split("<")[0][:60]
    tot[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
allt = sum(tot.values())
for k in sorted(tot, key=tot.get, reverse=True):
    print(f"{tot[k] / 1e3:10.1f} us {cnt[k]:5d}  {100 * tot[k] / allt:5.1f}%  {k}")
print(f"{allt / 1e3:10.1f} us total, {len(launches)} launches")
