"""Top stall-sampled SASS lines of an ncu report's source page:
python tools/ncu_hot.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
si, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
val = lambda r: int(r[si]) if r[si].isdigit() else 0  # noqa: E731
tot = sum(val(r) for r in data)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print("total samples", tot)
for i in sorted(sorted(range(len(data)), key=lambda i: -val(data[i]))[:n]):
    r = data[i]
    print(f"{i:5d} {val(r):6d} {r[ei]:>8s}  {r[1].strip()[:80]}")
