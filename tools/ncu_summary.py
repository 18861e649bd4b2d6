"""Summarise an `ncu --set full` report into profiles/ (text + traffic JSON).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep <config> profiles/rNN_ncu_<config>.txt
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

rep, config, out = sys.argv[1], sys.argv[2], Path(sys.argv[3])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
     "launch__grid_size", "launch__block_size", "smsp__issue_active.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
lines = [f"ncu --set full summary, config {config}, report {Path(rep).name}",
         "kernel | dur_us | dram_rd_MB | dram_wr_MB | dram% | sm% | issue% | warp_inst_M | occ% | regs | grid x block"]
traffic = {}
for r in rows[2:]:
    def g(m):
        i = h.index(m)
        v = float(r[i].replace(",", "")) if r[i] else 0.0
        return v * SCALE.get(units[i], 1)
    name = r[h.index("Kernel Name")].replace("(anonymous namespace)::", "").split("(")[0]
    name = name.replace("void ", "").replace("sdqz::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    dur = g(M[0])
    rd, wr = g(M[1]), g(M[2])
    lines.append(f"{name} | {dur*1e6:.1f} | {rd/1e6:.1f} | {wr/1e6:.1f} | {g(M[3]):.1f} | {g(M[4]):.1f} | "
                 f"{g(M[10]):.1f} | {g(M[5])/1e6:.2f} | {g(M[6]):.1f} | {int(g(M[7]))} | "
                 f"{int(g(M[8]))} x {int(g(M[9]))}")
    base = name.split("<")[0]
    traffic.setdefault(base, rd + wr)
out.parent.mkdir(parents=True, exist_ok=True)
out.write_text("\n".join(lines) + "\n")
tj = out.parent / "ncu_traffic.json"
allt = json.loads(tj.read_text()) if tj.exists() else {}
allt.setdefault(config, {}).update({k: int(v) for k, v in traffic.items()})
tj.write_text(json.dumps(allt, indent=1, sort_keys=True) + "\n")
print("\n".join(lines))
