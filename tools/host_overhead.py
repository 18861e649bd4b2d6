"""Wall-clock vs device time of the plan calls (host overhead per compress/decompress)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2007_09625_b200 import _lib  # noqa: E402
from paper_2007_09625_b200.pipeline import CompressPlan, DecompressPlan  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "hurricane"]
d = bench.device_field(cfg["dims"], 1)
plan = CompressPlan(d, cfg["dims"], eb=cfg["eb"], mode=cfg["mode"])
dev = plan.run()
dplan = DecompressPlan(dev)
for _ in range(3):
    plan.run()
    dplan.run()
torch.cuda.synchronize()
for name, fn in (("compress", plan.run), ("decompress", dplan.run)):
    ts, gs = [], []
    for _ in range(20):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        gs.append(a.elapsed_time(b) / 1e3)
    ts.sort()
    gs.sort()
    print(f"{name:10s} wall {ts[10]*1e6:8.1f} us   events {gs[10]*1e6:8.1f} us")
ctx = _lib.context()
ctx.set_timing(True)
plan.run()
dplan.run()
print(ctx.kernel_times())
ctx.set_timing(False)
