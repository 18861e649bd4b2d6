"""Phase timing of the public host-buffer API (compress(np) -> bytes -> decompress -> np)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2007_09625_b200 as S  # noqa: E402
from paper_2007_09625_b200 import pipeline as P  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "hurricane"]
dims = cfg["dims"]
h, pinned = bench.host_field(dims, 1)
h = h.reshape(dims)
pageable = np.array(h) if h.size < 1e9 else h


def t(label, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{label:40s} {min(ts)*1e3:9.3f} ms  (median {sorted(ts)[len(ts)//2]*1e3:9.3f})", flush=True)
    return r


blob = t("compress(pinned) -> bytes", lambda: S.compress(h, eb=cfg["eb"], mode=cfg["mode"]))
if h.size < 1e9: t("compress(pageable) -> bytes", lambda: S.compress(pageable, eb=cfg["eb"], mode=cfg["mode"]))
dev = t("compress_device(pinned)", lambda: P.compress_device(h, eb=cfg["eb"], mode=cfg["mode"]))
t("  to_device only", lambda: P._device.to_device(h))
t("  archive to_bytes", lambda: dev.to_bytes())
t("decompress(bytes) -> np", lambda: S.decompress(blob))
o = t("decompress_device(bytes)", lambda: P.decompress_device(blob))
t("  out.cpu().numpy()", lambda: o.cpu().numpy())
po = torch.empty(o.numel(), dtype=o.dtype, pin_memory=True)
t("  out -> pinned copy_", lambda: po.copy_(o.reshape(-1)))
t("  np.empty + fill (page faults)", lambda: np.empty(o.numel(), np.float32).fill(0))
