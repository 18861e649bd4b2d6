"""Per-source-line warp instructions and average active threads per instruction
(divergence) of one kernel, from the ncu source page (cuda,sass)."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, lines = "?", None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0] or len(r) < len(hdr) - 5:
        continue
    try:
        w = float(r[hdr.index("Instructions Executed")] or 0)
        t = float(r[hdr.index("Thread Instructions Executed")] or 0)
    except ValueError:
        continue
    if w:
        lines.append((w, t, f"{fname}:{r[0]}", r[1].strip()[:80]))
tw = sum(x[0] for x in lines) or 1
tt = sum(x[1] for x in lines)
print(f"warp-inst {tw/1e6:.2f}M thread-inst {tt/1e6:.1f}M avg active threads {tt/tw:.1f}")
for w, t, loc, src in sorted(lines, key=lambda x: -x[0])[:top]:
    print(f"{100*w/tw:5.1f}% inst {t/w:5.1f} thr  {loc:18s} {src}")
