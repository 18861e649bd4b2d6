"""Quick per-kernel timing of one config (device-generated field; timing only).

    python tools/kbench.py [config ...]   (hurricane cesm hacc nyx large)
"""
import json
import math
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2007_09625_b200 import _lib, synthetic  # noqa: E402
from paper_2007_09625_b200.pipeline import CompressPlan, DecompressPlan  # noqa: E402


def device_field(dims, seed=1):
    rows = dims[0]
    step = max(1, int(2**28 // max(1, math.prod(dims[1:]))))
    out = torch.empty(dims, dtype=torch.float32, device="cuda")
    for r0 in range(0, rows, step):
        r1 = min(rows, r0 + step)
        out[r0:r1] = synthetic.smooth_field_device(dims, seed, rows=(r0, r1), dtype=torch.float32)
    return out.reshape(-1)


def run(name, reps=10):
    cfg = bench.CONFIGS[name]
    d = device_field(cfg["dims"])
    plan = CompressPlan(d, cfg["dims"], eb=cfg["eb"], mode=cfg["mode"])
    dev = plan.run()
    dp = DecompressPlan(dev)
    for _ in range(3):
        dp.run(plan.run())
    flush = torch.empty(1 << 27, device="cuda")
    c_ms, d_ms = [], []
    for _ in range(reps):
        flush.zero_()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record()
        dv = plan.run()
        b.record()
        dp.run(dv)
        c.record()
        torch.cuda.synchronize()
        c_ms.append(a.elapsed_time(b))
        d_ms.append(b.elapsed_time(c))
    ctx = _lib.context()
    ctx.set_timing(True)
    for _ in range(reps):
        flush.zero_()
        dp.run(plan.run())
    torch.cuda.synchronize()
    kt = {k: round(v / reps, 4) for k, v in ctx.kernel_times().items() if not k.startswith("(")}
    ctx.set_timing(False)
    n = math.prod(cfg["dims"])
    tc, td = statistics.median(c_ms), statistics.median(d_ms)
    print(json.dumps({"config": name, "compress_ms": round(tc, 4), "decompress_ms": round(td, 4),
                      "gbs": round(4 * n / ((tc + td) / 1e3) / 1e9, 1),
                      "kernels": dict(sorted(kt.items(), key=lambda x: -x[1]))}), flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or ["hurricane"]:
        run(name)
