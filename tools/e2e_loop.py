"""Per-iteration phase times of the bench's end-to-end loop (compress(np) -> bytes,
decompress(bytes) -> np), to find where the wall-clock variance comes from."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2007_09625_b200 as S  # noqa: E402
from paper_2007_09625_b200 import pipeline as P  # noqa: E402
from paper_2007_09625_b200 import _device  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "hurricane"]
dims = cfg["dims"]
h, pinned = bench.host_field("x", dims, 1)
h = h.reshape(dims)
kw = dict(eb=cfg["eb"], mode=cfg["mode"])
for _ in range(3):
    S.decompress(S.compress(h, **kw))
torch.cuda.synchronize()
for it in range(10):
    t0 = time.perf_counter()
    dev = P.compress_device(h, **kw)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    blob = dev.to_bytes()
    t2 = time.perf_counter()
    o = P.decompress_device(blob)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    rec = _device.download(o)
    t4 = time.perf_counter()
    del rec
    print(f"it {it}: compress_device {1e3*(t1-t0):7.3f}  to_bytes {1e3*(t2-t1):7.3f}  "
          f"decompress_device {1e3*(t3-t2):7.3f}  download {1e3*(t4-t3):7.3f}  total {1e3*(t4-t0):7.3f} ms",
          flush=True)
