"""Per-CUDA-source-line stall samples / instructions of one kernel (ncu report,
source page in cuda,sass mode: SASS rows are attributed to the preceding line)."""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
fname, line, hdr = "?", None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:
        line = (fname, r[0])
        agg[line][2] = r[1].strip()
        continue
    if line is None:
        continue
    try:
        agg[line][0] += float(r[4] or 0)
        agg[line][1] += float(r[7] or 0)
    except (ValueError, IndexError):
        pass
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"samples {ts:.0f} warp-instructions {ti/1e6:.2f}M")
for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{s/ts*100:5.1f}% smp {i/ti*100:5.1f}% ins  {f}:{ln:5s} {src[:78]}")
