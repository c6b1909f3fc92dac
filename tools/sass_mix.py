"""Executed warp-instructions per SASS opcode from an ncu report's source page.
    python tools/sass_mix.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
si, ei = h.index("Source"), h.index("Instructions Executed")
c = Counter()
for r in rows[hdr + 1:]:
    if len(r) <= ei or not r[ei].isdigit():
        continue
    op = r[si].split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    c[o.split(".")[0]] += int(r[ei])
tot = sum(c.values())
for o, v in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{o:10s} {v:14d} {100 * v / tot:6.2f}%")
print("total", tot)
