"""Summarise an ncu report's SASS source page: instructions per opcode normalised
by a unit count, top stall lines.  usage: ncu_src.py report.ncu-rep units"""
import collections
import csv
import io
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ia = hdr.index("Instructions Executed")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
tot = sum(int(r[ia]) for r in data)
ts = sum(int(r[isamp]) for r in data)
print(f"instructions {tot}  per unit {tot / units:.1f}  stall samples {ts}")
byop = collections.Counter()
for r in data:
    s = r[src].strip().split()
    if not s:
        continue
    op = s[1] if s[0].startswith("@") else s[0]
    byop[op.split(".")[0]] += int(r[ia])
print(" ".join(f"{k}:{v / units:.1f}" for k, v in byop.most_common(24)))
print("top stall lines:")
for i, r in sorted(enumerate(data), key=lambda x: -int(x[1][isamp]))[:25]:
    print(f"  {i:5d} ex={int(r[ia]):9d} st={int(r[isamp]) / ts * 100:5.2f}% {r[src].strip()[:70]}")
