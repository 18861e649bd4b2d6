import sys; sys.path.insert(0, '.')
import torch, bench
from paper_2007_09625_b200.pipeline import CompressPlan, DecompressPlan
for name in sys.argv[1:]:
    cfg = bench.CONFIGS[name]
    d = bench.device_field(cfg["dims"], 1)
    plan = CompressPlan(d, cfg["dims"], eb=cfg["eb"], mode=cfg["mode"])
    dev = plan.run(); dp = DecompressPlan(dev)
    for _ in range(3): dp.run()
    torch.cuda.synchronize()
