#!/usr/bin/env python
"""Benchmark of the sdqz compress + decompress path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config hurricane|cesm|hacc|nyx|large] [--no-cpu-baseline]

One step = compress + decompress of one synthetic fp32 field of the config's
shape (reference metric: "compress & decompress GB/s (fp32 in)").  `value` is
whole-job fp32-input GB/s with the field resident in HBM (device-timed with
CUDA events, L2 flushed between steps); `e2e` is the same metric through the
public API with host buffers (pinned host field -> archive bytes -> host
field).  Under torchrun each rank processes its own field (weak scaling).
`--impl reference` times the CPU reference path (the oracle port of the
reference package, oracle/sdqz_oracle.py) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "cesm": dict(dims=(1800, 3600), eb=1e-4, mode="valrel", desc="2D CESM-ATM-shaped 1800x3600"),
    "hurricane": dict(dims=(100, 500, 500), eb=1e-4, mode="valrel",
                      desc="3D Hurricane-Isabel-shaped 100x500x500"),
    "hacc": dict(dims=(280953867,), eb=1e-4, mode="valrel", desc="1D HACC-shaped 280,953,867"),
    "nyx": dict(dims=(512, 512, 512), eb=1e-4, mode="valrel", desc="3D Nyx-shaped 512^3"),
    "large": dict(dims=(2048, 2048, 1024), eb=1e-4, mode="valrel",
                  desc="3D 2048x2048x1024 (17.2 GB fp32)"),
}
METRIC = "compress & decompress GB/s (fp32 in)"
L2_FLUSH_BYTES = 512 << 20


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# --------------------------------------------------------------------------
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------
# data
# --------------------------------------------------------------------------
def host_field(cfg_name: str, dims, seed: int, rank: int = 0):
    """Synthetic smooth field (reference synthetic.py profile) as a pinned host array."""
    import torch
    from paper_2007_09625_b200 import synthetic
    n = math.prod(dims)
    pinned = torch.empty(n, dtype=torch.float32, pin_memory=True)
    arr = pinned.numpy()
    if n <= 300_000_000:
        arr[:] = synthetic.smooth_rows(dims, seed).astype(np.float32).reshape(-1)
    else:   # slab-wise on the device (host f64 temporaries would not fit)
        dev = synthetic.smooth_field_device(dims, seed, dtype=torch.float32)
        pinned.copy_(dev.reshape(-1))
        del dev
    return arr, pinned


def device_field(dims, seed: int):
    import torch
    from paper_2007_09625_b200 import synthetic
    rows = dims[0]
    step = max(1, int(2**28 // max(1, math.prod(dims[1:]))))   # <= 2 GiB f64 temporaries
    out = torch.empty(dims, dtype=torch.float32, device="cuda")
    for r0 in range(0, rows, step):
        r1 = min(rows, r0 + step)
        out[r0:r1] = synthetic.smooth_field_device(dims, seed, rows=(r0, r1), dtype=torch.float32)
    return out.reshape(-1)


# --------------------------------------------------------------------------
# reference arm (CPU)
# --------------------------------------------------------------------------
def reference_arm(args, cfg, world, rank):
    if rank != 0:
        return 0
    from oracle import sdqz_oracle as O
    from paper_2007_09625_b200 import synthetic
    dims = cfg["dims"]
    # bounded sample: leading rows of the same field (~6e6 points)
    rows = max(1, min(dims[0], int(math.ceil(6e6 / max(1, math.prod(dims[1:]))))))
    sdims = (rows,) + tuple(dims[1:])
    data = synthetic.smooth_rows(dims, 1, (0, rows)).astype(np.float32)
    if len(dims) == 1:
        data = data[:rows]
    n = data.size
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        O.decompress(O.compress(data, sdims, eb=cfg["eb"], mode=cfg["mode"]), workers=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        blob = O.compress(data, sdims, eb=cfg["eb"], mode=cfg["mode"])
        O.decompress(blob, workers=cores)
    dt = time.perf_counter() - t0
    value = 4 * n * args.steps / dt / 1e9
    sample = f"rows [0,{rows}) of the {cfg['desc']} field ({n} points) per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": args.config, "dims": list(dims),
                                        "eb": cfg["eb"], "mode": cfg["mode"], "sample_dims": list(sdims)},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(data, dims, cfg):
    """Oracle port, one thread, on a bounded sample of the same field."""
    from oracle import sdqz_oracle as O
    # up to 2.5e7 points: the whole Hurricane workload (~5-10 s of one core)
    rows = max(1, min(dims[0], int(math.ceil(2.5e7 / max(1, math.prod(dims[1:]))))))
    sdims = (rows,) + tuple(dims[1:])
    sample = data.reshape(dims)[:rows].copy()
    t0 = time.perf_counter()
    blob = O.compress(sample, sdims, eb=cfg["eb"], mode=cfg["mode"])
    O.decompress(blob, workers=1)
    dt = time.perf_counter() - t0
    return {"value": 4 * sample.size / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"rows [0,{rows}) of the field ({sample.size} points), compress+decompress, "
                      f"oracle/sdqz_oracle.py (numpy port of the reference), 1 step"}


# --------------------------------------------------------------------------
# roofline bookkeeping
# --------------------------------------------------------------------------
def algorithmic_bytes(kernel: str, n: int, k: int, c: int, p: int) -> int | None:
    """Bytes a kernel must move per launch: N points, K
    outliers, C chunks, P payload bytes; u16 codes, fp32 field."""
    table = {
        "describe_kernel": 4 * n,                          # field read
        "dq3d_tma_kernel": 4 * n + 2 * n,                  # field read, codes written
        "dq": 4 * n + 2 * n,
        "chunk_stats_kernel": 2 * n + 4 * c,               # codes read, chunk bits written
        "chunk_pack32_kernel": 2 * n + p + 20 * k + 12 * c,  # codes, payload, outliers (+ input reads)
        "chunk_pack_kernel": 2 * n + p + 20 * k + 12 * c,
        "inflate_fast_kernel": p + 12 * c + 2 * n,         # payload, chunk bits + offsets, codes written
        "rq3d_block_kernel": 2 * n + 4 * n + 8 * k,        # codes read, field written, outlier values
        "rq2d_kernel": 2 * n + 4 * n + 8 * k,
        "rq2d_vec_kernel": 2 * n + 4 * n + 8 * k,
        "rq1d_kernel": 2 * n + 4 * n + 8 * k,
        "rq1d_vec_kernel": 2 * n + 4 * n + 8 * k,
        "rq1d_rec_kernel": 2 * n + 4 * n + 16 * k,         # codes read, field written, outlier records
        "outlier_check_kernel": 16 * k,
        "outlier_scatter_kernel": 16 * k + 8 * k + 2 * k,
    }
    for key, v in table.items():
        if kernel.startswith(key):
            return v
    return None


def load_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback"


def load_traffic(config: str, kernel: str):
    """dram read+write bytes per launch from the committed ncu --set full
    capture (profiles/ncu_traffic.json, tools/ncu_summary.py)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        t = json.loads(p.read_text()).get(config, {})
    except (OSError, ValueError):
        return None
    for name, v in t.items():
        if name == kernel or name.startswith(kernel) or kernel.startswith(name):
            return v
    return None


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def ours_arm(args, cfg, world, rank, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2007_09625_b200 as S
    from paper_2007_09625_b200 import _lib
    from paper_2007_09625_b200.pipeline import CompressPlan, DecompressPlan

    torch.cuda.set_device(local_rank)
    dims = cfg["dims"]
    n = math.prod(dims)
    seed = 1 + rank
    if args.config == "large":
        d_in = device_field(dims, seed)
        h_in, h_pinned = None, None
    else:
        h_in, h_pinned = host_field(args.config, dims, seed, rank)
        d_in = torch.from_numpy(h_in).cuda()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    ctx = _lib.context()

    plan = CompressPlan(d_in, dims, eb=cfg["eb"], mode=cfg["mode"])
    dev = plan.run()
    dplan = DecompressPlan(dev)

    def step():
        plan.run()
        dplan.run()

    for _ in range(max(args.warmup, 1)):
        step()
    hdr = plan.hdr
    K, C, P = int(hdr.n_outliers), int(hdr.n_chunks), int(hdr.payload_bytes)
    archive_bytes = hdr.total_bytes
    # correctness guard on the measured data: the error bound holds
    out = dplan.run().reshape(-1)
    q = S.quality(d_in, out)   # one native fp64 pass (no field-sized temporaries)
    err = q.max_abs_error
    amax = max(abs(float(d_in.min())), abs(float(d_in.max())))
    assert err <= hdr.eb_resolved * (1 + 1e-9) + 2 * np.spacing(np.float32(amax)), err

    stream = torch.cuda.current_stream()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0, replays0 = ctx.launches, ctx.graph_replays
    with Clocks(local_rank) as clk:
        for i in range(args.steps):
            flush.zero_()                       # evict the field/archive from L2
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = ctx.launches - launches0
    replays = ctx.graph_replays - replays0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t_local = sum(step_ms) / 1e3
    t = torch.tensor([t_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    value = world * 4 * n * args.steps / t_max / 1e9

    # split compress / decompress and per-kernel shares (probe pass, same events API)
    ctx.set_timing(True)
    probe = max(3, min(args.steps, 10))
    c_ms, d_ms = [], []
    for _ in range(probe):
        flush.zero_()
        a, b, c2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(stream)
        plan.run()
        b.record(stream)
        dplan.run()
        c2.record(stream)
        torch.cuda.synchronize()
        c_ms.append(a.elapsed_time(b))
        d_ms.append(b.elapsed_time(c2))
    ktimes = {k: v / probe for k, v in ctx.kernel_times().items()}
    ctx.set_timing(False)
    kernels = {k: v for k, v in ktimes.items() if not k.startswith("(") and k != "status_readback"}
    # roofline kernel: the largest one the bytes table covers (tiny bookkeeping
    # kernels have no byte-bound roofline)
    covered = {k: v for k, v in kernels.items() if algorithmic_bytes(k, n, K, C, P)}
    dom = max(covered or kernels, key=(covered or kernels).get)
    peak, peak_kind = load_peak()
    abytes = algorithmic_bytes(dom, n, K, C, P)
    achieved = abytes / (kernels[dom] / 1e3) / 1e9 if abytes else None

    # e2e through the public API with host buffers
    e2e_steps = max(5, min(args.steps, 10))
    e2e = None
    if h_in is not None:
        # three warm-up round trips: graph capture of both pipelines, the second result buffer of the pinned pool
        # (the previous result is still alive when the next one is allocated)
        for _ in range(3):
            blob = S.compress(h_in.reshape(dims), eb=cfg["eb"], mode=cfg["mode"])
            rec = S.decompress(blob)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            blob = S.compress(h_in.reshape(dims), eb=cfg["eb"], mode=cfg["mode"])
            rec = S.decompress(blob)
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        te_t = torch.tensor([te], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te_t, op=dist.ReduceOp.MAX)
        te = float(te_t.item())
        assert rec.shape == tuple(dims)
        e2e = {"value": world * 4 * n * e2e_steps / te / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": 4 * n + len(blob), "d2h_bytes_per_step": len(blob) + 4 * n,
               "steps": e2e_steps, "timing": "wall clock, cuda synchronize on both sides",
               "api": "paper_2007_09625_b200.compress(pinned np.ndarray) -> bytes; "
                      "decompress(bytes) -> np.ndarray"}

    base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and h_in is not None:
        base = cpu_baseline(h_in, dims, cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "dims": list(dims),
                       "eb": cfg["eb"], "mode": cfg["mode"], "cap": 1024,
                       "profile": "smooth (reference synthetic.py), seed 1+rank, fp32",
                       "l2": "flushed between steps (512 MiB write); per-step CUDA events",
                       "per_rank_points": n, "parallelism": f"replicas x{world}" if world > 1 else "1 GPU"},
            "compress_gbs": 4 * n / (statistics.median(c_ms) / 1e3) / 1e9,
            "decompress_gbs": 4 * n / (statistics.median(d_ms) / 1e3) / 1e9,
            "compression_ratio": 4 * n / archive_bytes,
            "archive": {"bytes": archive_bytes, "n_outliers": K, "n_chunks": C, "payload_bytes": P,
                        "max_abs_err_over_eb": err / hdr.eb_resolved},
            "kernel_ms": {k: round(v, 5) for k, v in sorted(kernels.items(), key=lambda x: -x[1])},
            "roofline": {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None,
                         "algorithmic_bytes": abytes, "ms": kernels[dom],
                         "traffic": load_traffic(args.config, dom)},
            "kernel_roofline": {
                kname: {"ms": round(kms, 5), "algorithmic_bytes": ab,
                        "gbs": round(ab / (kms / 1e3) / 1e9, 1),
                        "frac": round(ab / (kms / 1e3) / 1e9 / peak, 3)}
                for kname, kms in sorted(kernels.items(), key=lambda x: -x[1])
                if (ab := algorithmic_bytes(kname, n, K, C, P)) and kms > 0
                # a label whose launch skipped the work (e.g. the 64-bit-unit packer
                # when units are 32 bits, a 1D tail kernel) is not a roofline entry
                and ab / (kms / 1e3) / 1e9 <= 1.2 * peak
                and not (kname.startswith("chunk_pack_kernel") and int(hdr.unit_width) == 32)},
            "e2e": e2e,
            "gpu_launches": launches,
            "graph_replays": replays,
            "clocks": clk.summary(),
            "cpu_baseline": base,
        }
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="hurricane", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("note: warmup raised to 3")
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return reference_arm(args, cfg, world, rank)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return ours_arm(args, cfg, world, rank, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
