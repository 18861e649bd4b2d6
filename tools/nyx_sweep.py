"""BASELINE configs[3]: the Nyx-shaped 512^3 eb sweep (valrel 1e-2 .. 1e-5 x
smooth / sparse-near-zero, synthetic.py:25-60), one JSON line per point:
device compress / decompress GB/s (field resident in HBM, CUDA events, L2
flushed), CR, unit width, and the archive SHA-256 against the reference-run
archive (tests/golden/config_golden.json).

    python tools/nyx_sweep.py > profiles/r02_nyx_sweep.jsonl
"""
import hashlib
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2007_09625_b200 import synthetic  # noqa: E402
from paper_2007_09625_b200.pipeline import CompressPlan, DecompressPlan  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
GOLD = json.loads((ROOT / "tests" / "golden" / "config_golden.json").read_text())
DIMS = (512, 512, 512)
N = 512 ** 3


def main(reps=10):
    flush = torch.empty(1 << 27, device="cuda")
    for profile, key in (("smooth", "smooth"), ("sparse-near-zero", "sparse")):
        host = synthetic.generate_field(profile, DIMS, seed=1).astype(np.float32)
        d = torch.from_numpy(host.reshape(-1)).cuda()
        del host
        for eb in (1e-2, 1e-3, 1e-4, 1e-5):
            g = GOLD.get(f"nyx_{key}_{eb:.0e}")
            plan = CompressPlan(d, DIMS, eb=eb, mode="valrel")
            dev = plan.run()
            sha = hashlib.sha256(dev.to_bytes()).hexdigest()
            dp = DecompressPlan(dev)
            for _ in range(3):
                dp.run(plan.run())
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
            tc, td = statistics.median(c_ms), statistics.median(d_ms)
            h = dev.header
            print(json.dumps({
                "profile": profile, "eb": eb, "mode": "valrel", "dims": list(DIMS),
                "compress_gbs": round(4 * N / tc / 1e6, 1), "decompress_gbs": round(4 * N / td / 1e6, 1),
                "gbs": round(4 * N / (tc + td) / 1e6, 1), "cr": round(4 * N / h.total_bytes, 3),
                "unit_width": int(h.unit_width), "n_outliers": int(h.n_outliers),
                "archive_sha256": sha, "matches_reference": (sha == g["archive_sha256"]) if g else None}),
                flush=True)
        del d
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
