#!/usr/bin/env python
"""Benchmark of the sdqz compress + decompress path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config hurricane|cesm|hacc|nyx|large] [--no-cpu-baseline]

One step = compress + decompress of one synthetic fp32 field of the config's
shape (reference metric: "compress & decompress GB/s (fp32 in)").  `value` is
whole-job fp32-input GB/s with the field resident in HBM (device-timed with
CUDA events, L2 flushed between steps); `e2e` is the same metric through the
public API with host buffers (pinned host field -> archive bytes -> host
field).  Under torchrun (N > 1) the field is split into slabs of whole block
rows, one per rank, compressed into one sharded archive and decompressed in
place (strong scaling, paper_2007_09625_b200/sharded.py).  `--impl reference`
times the CPU reference path (the oracle port of the reference package,
oracle/sdqz_oracle.py) on the host cores.
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
    "cesm": dict(dims=(1800, 3600), eb=1e-4, mode="valrel", golden="cesm",
                 desc="2D CESM-ATM-shaped 1800x3600"),
    "hurricane": dict(dims=(100, 500, 500), eb=1e-4, mode="valrel", golden="hurricane",
                      desc="3D Hurricane-Isabel-shaped 100x500x500"),
    "hacc": dict(dims=(280953867,), eb=1e-4, mode="valrel", golden="hacc",
                 desc="1D HACC-shaped 280,953,867"),
    "nyx": dict(dims=(512, 512, 512), eb=1e-4, mode="valrel", golden="nyx_smooth_1e-04",
                desc="3D Nyx-shaped 512^3"),
    "large": dict(dims=(2048, 2048, 1024), eb=1e-4, mode="valrel", golden="large",
                  desc="3D 2048x2048x1024 (17.2 GB fp32), BASELINE.json configs[4]"),
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
def host_field(dims, seed: int):
    """The reference's smooth profile (synthetic.py:25-35), bit-identical to its
    generate_field, evaluated slab-wise on all host cores straight into pinned
    memory (the 17.2 GB config never materialises an f64 field)."""
    import torch
    from concurrent.futures import ThreadPoolExecutor
    from paper_2007_09625_b200 import synthetic
    n = math.prod(dims)
    pinned = torch.empty(n, dtype=torch.float32, pin_memory=True)
    arr = pinned.numpy()
    inner = math.prod(dims[1:])
    rows = max(1, min(dims[0], (1 << 24) // max(1, inner))) if len(dims) > 1 else dims[0]
    if len(dims) == 1:   # 1D: the whole axis at once (ufuncs release the GIL anyway)
        arr[:] = synthetic.smooth_rows(dims, seed).astype(np.float32)
        return arr, pinned

    def fill(r0):
        r1 = min(dims[0], r0 + rows)
        arr[r0 * inner:r1 * inner] = synthetic.smooth_rows(dims, seed, (r0, r1)).astype(np.float32).reshape(-1)

    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
        list(ex.map(fill, range(0, dims[0], rows)))
    return arr, pinned


def golden_for(config: str):
    """Reference archive hashes of this config (tests/golden/config_golden.json,
    made by running the reference in the build container)."""
    try:
        return json.loads((ROOT / "tests" / "golden" / "config_golden.json").read_text()).get(config)
    except (OSError, ValueError):
        return None


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# --------------------------------------------------------------------------
# CPU reference path (oracle port of the reference package, oracle/sdqz_oracle.py)
# --------------------------------------------------------------------------
def cpu_sample(cfg, max_points: float):
    """A bounded sample of the workload: the leading whole blocks of the field
    (rows along axis 0, then columns along axis 1 for 3D), compressed with the
    FULL field's resolved bound (abs mode) and chunk size so it quantizes and
    chunks exactly as the same points do inside the full-field archive."""
    from paper_2007_09625_b200 import synthetic
    from paper_2007_09625_b200.huffman import default_chunk_size
    dims = cfg["dims"]
    g = golden_for(cfg["golden"]) or {}
    eb = g.get("eb_resolved")
    if eb is None:
        f = synthetic.smooth_rows(dims, 1) if math.prod(dims) < 5e8 else None
        eb = cfg["eb"] * float(np.float32(f.max()) - np.float32(f.min())) if f is not None else cfg["eb"]
    b0 = {1: 32, 2: 16, 3: 8}[len(dims)]
    if len(dims) == 1:
        m = int(min(dims[0], max(b0, max_points // b0 * b0)))
        sdims = (m,)
        data = synthetic.smooth_rows(dims, 1, (0, m))
    else:
        inner = math.prod(dims[1:])
        rows = int(min(dims[0], max(b0, (max_points // inner) // b0 * b0)))
        cols = dims[1]
        if rows * inner > 1.5 * max_points and len(dims) == 3:   # one block row, fewer columns
            cols = int(min(dims[1], max(b0, (max_points // (rows * dims[2])) // b0 * b0)))
        sdims = (rows, cols) + tuple(dims[2:])
        data = synthetic.smooth_rows(dims, 1, (0, rows))[:, :cols]
    data = np.ascontiguousarray(data, dtype=np.float32)
    chunk = default_chunk_size(math.prod(dims))
    desc = (f"leading {'x'.join(map(str, sdims))} block-aligned box of the {cfg['desc']} field "
            f"({data.size} points), abs eb = the full field's resolved bound {eb:.6g}, chunk {chunk}; "
            f"throughput is per point, so it extrapolates linearly to the full field")
    return data, sdims, eb, chunk, desc


def time_cpu(data, sdims, eb, chunk, workers: int, steps: int = 1):
    from oracle import sdqz_oracle as O
    t0 = time.perf_counter()
    for _ in range(steps):
        blob = O.compress(data, sdims, eb=eb, mode="abs", chunk_size=chunk)
        O.decompress(blob, workers=workers)
    return (time.perf_counter() - t0) / steps


def reference_arm(args, cfg, world, rank):
    """The CPU reference path on the host cores (the oracle port: the reference
    is pure Python + numpy and is not importable on the GPU box)."""
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    # the reference's `workers` threads only its decode (numpy holds the GIL
    # elsewhere) and can be slower than one thread: probe both on a small
    # sample, then warm up and time the faster on the full ~8 M-point sample
    # (large enough that per-call fixed costs do not dominate)
    pdata, psdims, peb, pchunk, _ = cpu_sample(cfg, 1e6)
    w1 = time_cpu(pdata, psdims, peb, pchunk, 1)
    wn = time_cpu(pdata, psdims, peb, pchunk, cores)
    workers = cores if wn < w1 else 1
    data, sdims, eb, chunk, desc = cpu_sample(cfg, 8e6)
    time_cpu(data, sdims, eb, chunk, workers, steps=max(1, min(args.warmup, 2)))
    dt = time_cpu(data, sdims, eb, chunk, workers, steps=args.steps) * args.steps
    value = 4 * data.size * args.steps / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong" if args.config == "large" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "dims": list(cfg["dims"]), "eb": cfg["eb"],
                   "mode": cfg["mode"], "sample_dims": list(sdims)},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": workers, "kind": "port",
                         "cpu": cpu_model(), "host_cores": cores, "workers": workers,
                         "workers_choice": f"faster of workers=1 ({w1:.2f} s) and workers={cores} "
                                           f"({wn:.2f} s) on a 1 M-point probe of the same field",
                         "sample": desc + " (per step)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(cfg):
    """Oracle port on one core (workers=1), a ~10-20 s bounded sample."""
    data, sdims, eb, chunk, desc = cpu_sample(cfg, 8e6)
    dt = time_cpu(data, sdims, eb, chunk, 1)
    return {"value": 4 * data.size / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "port",
            "cpu": cpu_model(), "workers": 1,
            "sample": desc + "; compress + decompress, oracle/sdqz_oracle.py (numpy port of the "
                             "reference, same speed as the reference in the build container), 1 step"}


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
    import hashlib

    import torch
    import torch.distributed as dist

    import paper_2007_09625_b200 as S
    from paper_2007_09625_b200 import _lib
    from paper_2007_09625_b200.pipeline import CompressPlan, DecompressPlan

    torch.cuda.set_device(local_rank)
    dims = cfg["dims"]
    n = math.prod(dims)
    seed = 1 + rank
    t0 = time.perf_counter()
    h_in, h_pinned = host_field(dims, seed)
    log(f"field {dims} generated in {time.perf_counter() - t0:.1f} s")
    d_in = h_pinned.cuda()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    ctx = _lib.context()

    plan = CompressPlan(d_in, dims, eb=cfg["eb"], mode=cfg["mode"])
    dev = plan.run()
    dplan = DecompressPlan(dev)

    def step():
        dplan.run(plan.run())

    for _ in range(max(args.warmup, 1)):
        step()
    dev = plan.run()
    hdr = dev.header
    K, C, P = int(hdr.n_outliers), int(hdr.n_chunks), int(hdr.payload_bytes)
    archive_bytes = hdr.total_bytes
    # parity guard on the measured data: the archive is the reference's (SHA-256
    # of the reference-run archive, tests/golden/config_golden.json) and the
    # error bound holds
    golden = golden_for(cfg["golden"]) if seed == 1 else None
    sha = hashlib.sha256(dev.to_bytes()).hexdigest()
    matches = (sha == golden["archive_sha256"]) if golden else None
    out = dplan.run(dev).reshape(-1)
    q = S.quality(d_in, out)   # one native fp64 pass (no field-sized temporaries)
    err = q.max_abs_error
    amax = max(abs(float(d_in.min())), abs(float(d_in.max())))
    assert err <= hdr.eb_resolved * (1 + 1e-9) + 2 * np.spacing(np.float32(amax)), err
    del out

    stream = torch.cuda.current_stream()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0, replays0 = ctx.launches, ctx.graph_replays
    with Clocks(local_rank) as clk:
        for i in range(args.steps):
            flush.zero_()                       # evict the field/archive from L2
            ev[i][0].record(stream)
            d = plan.run()
            ev[i][1].record(stream)             # compress / decompress split (no timers)
            dplan.run(d)
            ev[i][2].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = ctx.launches - launches0
    replays = ctx.graph_replays - replays0
    step_ms = [a.elapsed_time(c) for a, b, c in ev]
    c_ms = [a.elapsed_time(b) for a, b, c in ev]
    d_ms = [b.elapsed_time(c) for a, b, c in ev]
    t_local = sum(step_ms) / 1e3
    t = torch.tensor([t_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    value = world * 4 * n * args.steps / t_max / 1e9

    # per-kernel device times (separate probe pass: the context's event timer
    # marks every launch, which turns graph replay off)
    ctx.set_timing(True)
    probe = max(3, min(args.steps, 10))
    for _ in range(probe):
        flush.zero_()
        dplan.run(plan.run())
    torch.cuda.synchronize()
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
    tc, td = statistics.median(c_ms) / 1e3, statistics.median(d_ms) / 1e3
    comp_bytes = (12 if cfg["mode"] == "valrel" else 8) * n + P + 16 * K + 4 * C
    decomp_bytes = 8 * n + P + 16 * K + 4 * C

    # e2e through the public API with host buffers: pinned host field ->
    # compress() -> archive bytes -> decompress() -> host field, every step
    e2e_steps = max(3, min(args.steps, 5 if n > 1e9 else 10))
    # each step drops the previous result before decompressing (a user keeping
    # every 17 GB result alive would also pay a fresh page-locked allocation)
    rec = None
    for _ in range(2):   # graph capture of both pipelines, pinned result pool
        blob = S.compress(h_in.reshape(dims), eb=cfg["eb"], mode=cfg["mode"])
        rec = None
        rec = S.decompress(blob)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        blob = S.compress(h_in.reshape(dims), eb=cfg["eb"], mode=cfg["mode"])
        rec = None
        rec = S.decompress(blob)
    torch.cuda.synchronize()
    te = time.perf_counter() - t0
    te_t = torch.tensor([te], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te_t, op=dist.ReduceOp.MAX)
    te = float(te_t.item())
    assert rec.shape == tuple(dims) and len(blob) == archive_bytes
    e2e = {"value": world * 4 * n * e2e_steps / te / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": 4 * n + len(blob), "d2h_bytes_per_step": len(blob) + 4 * n,
           "steps": e2e_steps, "timing": "wall clock, cuda synchronize on both sides",
           "api": "paper_2007_09625_b200.compress(pinned np.ndarray) -> bytes; "
                  "decompress(bytes) -> np.ndarray"}
    del rec, blob

    base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        base = cpu_baseline(cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "dims": list(dims),
                       "eb": cfg["eb"], "mode": cfg["mode"], "cap": 1024,
                       "profile": "smooth (reference synthetic.py), seed 1+rank, fp32, bit-identical "
                                  "to the reference's generate_field",
                       "l2": "flushed between steps (512 MiB write); per-step CUDA events",
                       "per_rank_points": n,
                       "parallelism": f"replicas x{world}" if world > 1 else "1 GPU"},
            "compress_gbs": 4 * n / tc / 1e9,
            "decompress_gbs": 4 * n / td / 1e9,
            "compression_ratio": 4 * n / archive_bytes,
            "parity": {"archive_sha256": sha, "reference_sha256": golden["archive_sha256"] if golden else None,
                       "archive_matches_reference": matches,
                       "max_abs_err_over_eb": err / hdr.eb_resolved},
            "archive": {"bytes": archive_bytes, "n_outliers": K, "n_chunks": C, "payload_bytes": P},
            "pipeline_roofline": {
                "compress": {"algorithmic_bytes": comp_bytes, "ms": tc * 1e3,
                             "gbs": comp_bytes / tc / 1e9, "frac": comp_bytes / tc / 1e9 / peak},
                "decompress": {"algorithmic_bytes": decomp_bytes, "ms": td * 1e3,
                               "gbs": decomp_bytes / td / 1e9, "frac": decomp_bytes / td / 1e9 / peak},
                "bytes": "compress 12N+P+16K+4C (valrel), decompress 8N+P+16K+4C (SURVEY.md 8d)"},
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


def sharded_arm(args, cfg, world, rank, local_rank):
    """N > 1: the config's field split into slabs of whole block rows over the
    ranks (strong scaling: the field is fixed, each rank holds 1/N of it),
    compressed into one ShardedArchive and decompressed in place
    (paper_2007_09625_b200.sharded)."""
    import hashlib

    import torch
    import torch.distributed as dist

    from paper_2007_09625_b200 import _lib, sharded, synthetic
    from paper_2007_09625_b200.core import QuantConfig

    dims = cfg["dims"]
    n = math.prod(dims)
    inner = math.prod(dims[1:])
    b0 = QuantConfig.for_rank(1.0, len(dims)).block_shape[0]
    rows = sharded.slab_rows(dims[0], b0, world)
    r0 = sum(rows[:rank])
    n_local = rows[rank] * inner
    # this rank's slab of the reference's smooth field (bit-identical rows)
    t0 = time.perf_counter()
    pinned = torch.empty(max(n_local, 1), dtype=torch.float32, pin_memory=True)
    arr = pinned.numpy()
    step_rows = max(1, (1 << 24) // max(1, inner))
    from concurrent.futures import ThreadPoolExecutor

    def fill(a):
        b = min(rows[rank], a + step_rows)
        arr[a * inner:b * inner] = synthetic.smooth_rows(dims, 1, (r0 + a, r0 + b)).astype(np.float32).reshape(-1)

    with ThreadPoolExecutor(max_workers=max(1, min(16, (os.cpu_count() or 1) // world))) as ex:
        list(ex.map(fill, range(0, rows[rank], step_rows)))
    local_dims = (rows[rank],) + tuple(dims[1:])
    d_in = pinned[:n_local].cuda().view(local_dims)
    log(f"rank {rank}: slab rows [{r0}, {r0 + rows[rank]}) generated in {time.perf_counter() - t0:.1f} s")
    ctx = _lib.context()
    kw = dict(eb=cfg["eb"], mode=cfg["mode"])

    def step():
        ar = sharded.compress_sharded_device(d_in, dims, **kw)
        out = sharded.decompress_sharded(ar, device=True)
        return ar, out

    for _ in range(max(args.warmup, 1)):
        ar, out = step()
    # parity guard: the assembled archive is the reference's (gathered once,
    # outside the timed region), and the slab's error bound holds
    golden = golden_for(cfg["golden"])
    blob = ar.gather(root=0)
    sha = hashlib.sha256(blob).hexdigest() if blob is not None else None
    del blob
    import paper_2007_09625_b200 as S
    err = S.quality(d_in.reshape(-1), out.reshape(-1)).max_abs_error if n_local else 0.0
    assert err <= ar.header.eb_resolved * (1 + 1e-9) + 2 * np.spacing(np.float32(8)), err
    del out
    stream = torch.cuda.current_stream()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    with Clocks(torch.cuda.current_device()) as clk:
        for i in range(args.steps):
            ev[i][0].record(stream)
            ar = sharded.compress_sharded_device(d_in, dims, **kw)
            ev[i][1].record(stream)
            out = sharded.decompress_sharded(ar, device=True)
            ev[i][2].record(stream)
            del out
        torch.cuda.synchronize()
    dist.barrier()
    launches = ctx.launches - launches0
    c_ms = [a.elapsed_time(b) for a, b, c in ev]
    d_ms = [b.elapsed_time(c) for a, b, c in ev]
    log(f"rank {rank}: compress ms per step {[round(x, 2) for x in c_ms]}, "
        f"decompress ms per step {[round(x, 2) for x in d_ms]}")
    tt = torch.tensor([sum(c_ms) + sum(d_ms), statistics.median(c_ms), statistics.median(d_ms)],
                      dtype=torch.float64)
    tt = tt.cuda() if dist.get_backend() == "nccl" else tt
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max, c_med, d_med = (float(x) for x in tt.cpu())
    value = 4 * n * args.steps / (t_max / 1e3) / 1e9

    # e2e through the public API with host buffers: this rank's pinned slab ->
    # device -> compress_sharded_device -> ShardedArchive.write (every rank
    # writes its own byte ranges of one archive file) -> decompress_sharded ->
    # host slab
    import shutil
    import tempfile
    # one archive file in RAM-backed /dev/shm when it has room, else the temp dir
    shm = "/dev/shm" if os.path.isdir("/dev/shm") and shutil.disk_usage("/dev/shm").free > 4 * 4 * n // 10 \
        else tempfile.gettempdir()
    path = os.environ.get("SDQZ_BENCH_ARCHIVE", os.path.join(shm, f"sdqz_bench_n{world}.sdqz"))
    host_out = torch.empty(max(n_local, 1), dtype=torch.float32, pin_memory=True)
    e2e_steps = max(2, min(args.steps, 3))
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        d = pinned[:n_local].cuda().view(local_dims)
        ar = sharded.compress_sharded_device(d, dims, **kw)
        nbytes = ar.write(path)
        o = sharded.decompress_sharded(ar, device=True)
        host_out[:n_local].copy_(o.reshape(-1))
        del d, o
    torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    te = te.cuda() if dist.get_backend() == "nccl" else te
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    te = float(te.cpu())
    my_bytes = 16 * int(ar.rank_sizes[rank, 2]) + 4 * int(ar.rank_sizes[rank, 0]) + int(ar.rank_sizes[rank, 1])
    if rank == 0:
        try:
            os.remove(path)
        except OSError:
            pass
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "dims": list(dims), "eb": cfg["eb"],
                       "mode": cfg["mode"], "cap": 1024,
                       "profile": "smooth (reference synthetic.py), seed 1, fp32, bit-identical slab rows",
                       "parallelism": f"{world} slabs of {rows[0]} rows (axis 0), one GPU each",
                       "collective_backend": dist.get_backend(),
                       "l2": "inputs larger than L2 (per-rank slab >= 2 GB)",
                       "per_rank_points": n_local},
            "compress_gbs": 4 * n / (c_med / 1e3) / 1e9,
            "decompress_gbs": 4 * n / (d_med / 1e3) / 1e9,
            "compression_ratio": 4 * n / ar.nbytes,
            "parity": {"archive_sha256": sha,
                       "reference_sha256": golden["archive_sha256"] if golden else None,
                       "archive_matches_reference": (sha == golden["archive_sha256"]) if golden else None,
                       "max_abs_err_over_eb (rank 0 slab)": err / ar.header.eb_resolved},
            "archive": {"bytes": ar.nbytes, "n_outliers": ar.header.n_outliers,
                        "n_chunks": ar.header.n_chunks, "payload_bytes": ar.header.payload_bytes},
            "e2e": {"value": 4 * n * e2e_steps / te / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": 4 * n_local, "d2h_bytes_per_step": my_bytes + 4 * n_local,
                    "steps": e2e_steps, "timing": "wall clock, max over ranks",
                    "api": "sharded.compress_sharded_device(pinned slab) -> ShardedArchive.write(path) "
                           "(parallel byte-range writes of one archive file); "
                           "decompress_sharded(archive) -> pinned host slab"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="large", choices=sorted(CONFIGS))
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
        ndev = torch.cuda.device_count()
        torch.cuda.set_device(local_rank % ndev)
        if ndev >= world and os.environ.get("SDQZ_BENCH_BACKEND", "nccl") == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:   # several ranks per GPU (tests on one GPU): gloo
            dist.init_process_group("gloo")
    try:
        if world > 1:
            return sharded_arm(args, cfg, world, rank, local_rank)
        return ours_arm(args, cfg, world, rank, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
