"""Decoder debugging: codes after a fused decompress vs the compressor's codes
(scratch slot S_CODES), first mismatching chunks with their geometry."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from kbench import device_field  # noqa: E402
from paper_2007_09625_b200 import _lib  # noqa: E402
from paper_2007_09625_b200.pipeline import CompressPlan, DecompressPlan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "hurricane"
cfg = bench.CONFIGS[name]
d = device_field(cfg["dims"], 1)
n = d.numel()
plan = CompressPlan(d, cfg["dims"], eb=cfg["eb"], mode=cfg["mode"])
dev = plan.run()
ctx = _lib.context()
want = np.zeros(n, np.uint16)
ctx.call("sdqz_debug_read", 0, ctypes.c_void_p(want.ctypes.data), want.nbytes)
try:
    DecompressPlan(dev).run()
    print("decompress ok")
except Exception as e:  # noqa: BLE001
    print("decompress error:", e)
got = np.zeros(n, np.uint16)
ctx.call("sdqz_debug_read", 0, ctypes.c_void_p(got.ctypes.data), got.nbytes)
h = dev.header
chunk = h.chunk_size
bad = np.flatnonzero(got != want)
print("mismatches", bad.size, "chunk", chunk, "n_chunks", h.n_chunks)
blob = dev.to_bytes()
from oracle import sdqz_oracle as O  # noqa: E402
p = O.unpack_archive(blob)
bits = np.asarray(p.chunk_bits, np.int64)
for c in np.unique(bad // chunk)[:6]:
    idx = bad[bad // chunk == c]
    B = int(bits[c]); cnt = min(chunk, n - c * chunk)
    print(f"chunk {c}: B={B} cnt={cnt} bpc={B / cnt:.2f} mism={idx.size} first={idx[0] - c * chunk} last={idx[-1] - c * chunk}")
    o = idx[0] - c * chunk
    print("   want", want[c * chunk + o - 3: c * chunk + o + 8])
    print("   got ", got[c * chunk + o - 3: c * chunk + o + 8])
