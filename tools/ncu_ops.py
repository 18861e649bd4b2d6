"""Opcode histogram (executed warp instructions) of one kernel in an ncu report."""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == 'Address')
h = rows[hi]
si, ii = h.index('Source'), h.index('Instructions Executed')
ops, seen = collections.Counter(), set()
for r in rows[hi + 1:]:
    if len(r) <= ii or r[0] in seen:
        continue
    seen.add(r[0])
    try:
        n = float(r[ii])
    except ValueError:
        continue
    src = r[si].strip().split()
    op = src[1] if src and src[0].startswith('@') else (src[0] if src else '?')
    ops[op.split('.')[0]] += n
tot = sum(ops.values())
print(f"total {tot/1e6:.2f}M warp instructions")
for k, v in ops.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 20):
    print(f"  {k:10s} {v/1e6:8.2f}M {v/tot*100:5.1f}%")
