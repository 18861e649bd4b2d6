"""Top SASS instructions by stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr_i]
si, ii, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
data = [r for r in rows[hdr_i + 1:] if len(r) > si and r[si].replace('.', '').isdigit()]
tot = sum(float(r[si]) for r in data) or 1
print("total samples", tot, "instructions", sum(float(r[ii] or 0) for r in data))
for r in sorted(data, key=lambda r: -float(r[si]))[:top]:
    top_st = sorted(((float(r[c] or 0), h[c][6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{float(r[si])/tot*100:5.1f}% {r[ii]:>9s}  {r[src].strip()[:70]:70s} {top_st}")
