"""Markdown results tables from profiles/<tag>_bench_*.json.

    python tools/results_table.py r02
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
names = [("large", "2048×2048×1024 (17.2 GB, BASELINE configs[4], bench default)"), ("hacc", "HACC 280,953,867 (1D)"),
         ("nyx", "Nyx 512³"), ("hurricane", "Hurricane 100×500×500"), ("cesm", "CESM 1800×3600 (2D)")]
rows, kr = [], []
for key, desc in names:
    p = ROOT / "profiles" / f"{tag}_bench_{key}.json"
    if not p.exists():
        continue
    d = json.loads(p.read_text().strip().splitlines()[-1])
    pr = d["pipeline_roofline"]
    rows.append(f"| {desc} | {d['value']:.0f} | {d['compress_gbs']:.0f} | {d['decompress_gbs']:.0f} | "
                f"{pr['compress']['frac'] * 100:.0f}% / {pr['decompress']['frac'] * 100:.0f}% | "
                f"{d['e2e']['value']:.1f} | {d['compression_ratio']:.2f} | "
                f"{'yes' if d['parity']['archive_matches_reference'] else 'no'} |")
    kk = d["kernel_roofline"]
    kr.append((key, {k: v["frac"] for k, v in kk.items()}, d["roofline"]))
print("| Workload (smooth profile, valrel 1e-4) | device GB/s (compress + decompress) | compress GB/s | "
      "decompress GB/s | pipeline HBM fraction (c / d) | e2e GB/s (host API) | CR | archive = reference run |")
print("|---|---|---|---|---|---|---|---|")
print("\n".join(rows))
print()
allk = []
for _, f, _ in kr:
    for k in f:
        if k not in allk:
            allk.append(k)
print("| Kernel | " + " | ".join(k for k, _, _ in kr) + " |")
print("|---|" + "---|" * len(kr))
for k in allk:
    print(f"| {k} | " + " | ".join(f"{f[k] * 100:.0f}%" if k in f else "—" for _, f, _ in kr) + " |")
print()
for key, _, r in kr:
    tr = r["traffic"]
    if tr is None:   # bench run before the config's ncu capture: take it from the committed file
        t = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text()).get(key, {})
        tr = next((v for k, v in t.items() if k.startswith(r["kernel"]) or r["kernel"].startswith(k)), None)
    trs = f"{tr / 1e9:.2f} GB" if tr else "n/a"
    print(f"* {key}: dominant kernel `{r['kernel']}` {r['achieved']:.0f} GB/s = {r['frac'] * 100:.1f}% of "
          f"{r['peak']:.0f} GB/s ({r['peak_kind']}); ncu DRAM traffic per launch {trs} vs "
          f"{r['algorithmic_bytes'] / 1e9:.2f} GB algorithmic")
