"""Key metrics of every kernel in an ncu report (details page)."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Issue Slots Busy", "Executed Ipc Active", "Achieved Occupancy",
        "Registers Per Thread", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block",
        "Executed Instructions", "Avg. Active Threads Per Warp", "Avg. Not Predicated Off Threads Per Warp",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Memory Throughput", "Compute (SM) Throughput",
        "Theoretical Occupancy", "Block Limit Shared Mem", "Block Limit Registers"]
rep = sys.argv[1]
extra = sys.argv[2:]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ki, mi, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
idi = hdr.index("ID")
cur = None
for r in rows[1:]:
    if len(r) <= vi:
        continue
    if r[idi] != cur:
        cur = r[idi]
        print(f"== [{cur}] {r[ki][:90]}")
    if r[mi] in KEYS or any(e in r[mi] for e in extra):
        print(f"   {r[mi]:45s} {r[vi]:>14s} {r[ui]}")
