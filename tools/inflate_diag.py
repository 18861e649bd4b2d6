"""Decompress a config field once and print the warp-decoder diagnostics."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2007_09625_b200 import _lib  # noqa: E402
from paper_2007_09625_b200.pipeline import CompressPlan, DecompressPlan  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "hurricane"]
d = bench.device_field(cfg["dims"], 1)
dev = CompressPlan(d, cfg["dims"], eb=cfg["eb"], mode=cfg["mode"]).run()
DecompressPlan(dev).run()
ctx = _lib.context()
out = (ctypes.c_uint64 * 3)()
ctx.lib.sdqz_debug_counters(ctx.h, out, 3)
print("chunks", dev.header.n_chunks, "lane redecodes", out[0], "unsynced chunks", out[1],
      "sequential chunks", out[2])
