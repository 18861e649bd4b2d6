"""Codebook phase timing + histogram shape for a config (debug build via SDQZ_LIB_PATH)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
sys.path.insert(0, str(Path(__file__).resolve().parent))
from kbench import device_field  # noqa: E402
import paper_2007_09625_b200 as S  # noqa: E402
from paper_2007_09625_b200.pipeline import CompressPlan  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "hurricane"]
d = device_field(cfg["dims"])
plan = CompressPlan(d, cfg["dims"], eb=cfg["eb"], mode=cfg["mode"])
for _ in range(3):
    dev = plan.run()
torch.cuda.synchronize()
blob = dev.to_bytes()
h = S.parse_header(blob)
bw = np.frombuffer(blob[S.HEADER_SIZE:S.HEADER_SIZE + h.cap], np.uint8)
print("present", int((bw > 0).sum()), "max_bw", int(bw.max()), "cap", h.cap)
