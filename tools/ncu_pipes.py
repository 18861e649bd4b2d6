"""Pipe utilisation (% of peak) per kernel from an ncu report: which
functional unit (fma / alu / fp64 / lsu / xu ...) bounds an issue-bound kernel.

    python tools/ncu_pipes.py report.ncu-rep [kernel-regex]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
ki = h.index("Kernel Name")
for r in rows[2:]:
    if pat and not pat.search(r[ki]):
        continue
    print(r[ki][:60])
    out = []
    for i, n in enumerate(h):
        if "pipe" in n and "pct_of_peak" in n and i < len(r):
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            if v >= 3:
                out.append((v, n))
    for v, n in sorted(out, reverse=True)[:14]:
        print(f"   {v:6.1f}  {n}")
