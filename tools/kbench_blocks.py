"""Compress / decompress device time for non-default block shapes (row f4).

    python tools/kbench_blocks.py            (Nyx-shaped 512^3, 2D 8192^2, 1D 2^28)
    python tools/kbench_blocks.py 8192,8192:8,8 512,512,512:4,4,4     (selected cases)
"""
import json
import math
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))

import torch  # noqa: E402

from kbench import device_field  # noqa: E402
from paper_2007_09625_b200 import _lib  # noqa: E402
from paper_2007_09625_b200.pipeline import CompressPlan, DecompressPlan  # noqa: E402

CASES = [
    ((512, 512, 512), None), ((512, 512, 512), (4, 4, 4)), ((512, 512, 512), (16, 16, 16)),
    ((512, 512, 512), (8, 8, 16)), ((512, 512, 512), (2, 8, 32)),
    ((8192, 8192), None), ((8192, 8192), (8, 8)), ((8192, 8192), (32, 32)), ((8192, 8192), (4, 64)),
    ((1 << 28,), None), ((1 << 28,), (64,)), ((1 << 28,), (256,)), ((1 << 28,), (16,)),
]


def run(dims, block, reps=5):
    d = device_field(dims)
    plan = CompressPlan(d, dims, eb=1e-4, mode="valrel", block_shape=block)
    dev = plan.run()
    dp = DecompressPlan(dev)
    for _ in range(2):
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
    flush.zero_()
    dp.run(plan.run())
    torch.cuda.synchronize()
    kt = {k: round(v, 4) for k, v in ctx.kernel_times().items() if not k.startswith("(") and v > 0.02}
    ctx.set_timing(False)
    n = math.prod(dims)
    tc, td = statistics.median(c_ms), statistics.median(d_ms)
    print(json.dumps({"dims": dims, "block": block, "compress_ms": round(tc, 3), "decompress_ms": round(td, 3),
                      "gbs": round(4 * n / ((tc + td) / 1e3) / 1e9, 1), "cr": round(4 * n / dev.nbytes, 2),
                      "kernels": dict(sorted(kt.items(), key=lambda x: -x[1]))}), flush=True)
    del d, plan, dev, dp
    torch.cuda.empty_cache()


if __name__ == "__main__":
    sel = [tuple(tuple(int(v) for v in p.split(",")) for p in a.split(":")) for a in sys.argv[1:]]
    for dims, block in sel or CASES:
        run(dims, block)
