"""Decompress a config field once and print the warp-decoder diagnostics."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import bench  # noqa: E402
from kbench import device_field  # noqa: E402
from paper_2007_09625_b200 import _lib  # noqa: E402
from paper_2007_09625_b200.pipeline import CompressPlan, DecompressPlan  # noqa: E402

for name in sys.argv[1:] or ["hurricane"]:
    cfg = bench.CONFIGS[name]
    d = device_field(cfg["dims"], 1)
    dev = CompressPlan(d, cfg["dims"], eb=cfg["eb"], mode=cfg["mode"]).run()
    ctx = _lib.context()
    DecompressPlan(dev).run()
    out = (ctypes.c_uint64 * 3)()
    ctx.lib.sdqz_debug_counters(ctx.h, out, 3)
    print(name, "chunks", dev.header.n_chunks, "lane redecodes", out[0] & 0xFFFFFFFF,
          "buffer overflows", out[0] >> 32, "handed back", out[1], "sequential chunks", out[2], flush=True)
    del d, dev
