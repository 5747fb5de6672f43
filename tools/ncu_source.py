"""Per-SASS-instruction counts and stall samples from an ncu report.
    python tools/ncu_source.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ia = hdr.index("Instructions Executed")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
tot = sum(int(r[ia]) for r in data)
ts = sum(int(r[isamp]) for r in data)
print("total warp instructions", tot, "stall samples", ts)
groups = collections.Counter()
for r in data:
    groups[int(r[ia])] += 1
print("execution-count classes (count: #instructions):",
      sorted(((k, v) for k, v in groups.items()), key=lambda kv: -kv[0] * kv[1])[:10])
print("--- listing (addr, inst, executed, samples)")
for r in data:
    if int(r[ia]) * 100 >= tot // 20000 or int(r[isamp]) > ts // 200:
        print(r[0][-5:], r[src][:74].ljust(74), r[ia].rjust(10), r[isamp].rjust(7))
