"""One compress + decompress of a config-shaped field, for ncu captures.

    ncu --set full -k regex:'dq3d|inflate' -c 4 python tools/profile_step.py hurricane
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import bench  # noqa: E402
sys.path.insert(0, str(Path(__file__).resolve().parent))
from paper_2007_09625_b200.pipeline import CompressPlan, DecompressPlan  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "hurricane"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = bench.CONFIGS[cfg_name]
from kbench import device_field  # noqa: E402
d = device_field(cfg["dims"], 1)
plan = CompressPlan(d, cfg["dims"], eb=cfg["eb"], mode=cfg["mode"])
for _ in range(reps):
    dev = plan.run()
    DecompressPlan(dev).run()
torch.cuda.synchronize()
print("ok", dev.nbytes)
