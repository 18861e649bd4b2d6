"""Config-scale golden hashes: run the REFERENCE on BASELINE.json's configs.

Run in the build container (where /root/reference exists; ~62 GB RAM, 8 cores):

    python tests/golden/make_config_golden.py [--only NAME ...] [--procs 7]

For every config it records, from the reference's own output:
  * the SHA-256 of the fp32 input field (so a test can first prove that the
    box regenerated the same field),
  * the SHA-256 of the archive bytes and of each archive section, and the
    header fields (eb_resolved as hex, outliers, chunks, payload, unit),
  * the SHA-256 of the decompressed fp32 field.

Configs 1-4 (CESM 1800x3600, Hurricane 100x500x500, HACC 280,953,867, the
Nyx 512^3 sweep valrel 1e-2..1e-5 x smooth / sparse-near-zero) run the
reference's `compress` / `decompress` on the whole field.

Config 5 (2048x2048x1024, 17.2 GB fp32) does not fit the reference's f64
temporaries in host memory, so it runs the reference's OWN row-slab
decomposition -- the code path `compress_field` / `reconstruct_field` take for
workers > 1 (dualquant.py:230-273, :299-332): `prequantize` + `_compress_region`
per slab of whole block rows with outlier indices offset by the slab start,
one `histogram` per slab summed, `build_tree` + `canonize` on the sum,
`encode` + `deflate` per chunk-aligned slab (chunks never share state,
huffman.py:219-225), `inflate` of each slab's chunk range and
`_reconstruct_region` of each slab with its `searchsorted` outlier sub-range.
The recipe is validated against the whole-field reference on Nyx 512^3 (same
archive SHA) before it is trusted at 17.2 GB.  Input / output hashes of the
large field are digests of per-16-row-slab SHA-256s (see `slab_digest`).

The field generator for slabs restates the reference's `_smooth`
(synthetic.py:25-35) with axis 0 sliced; it is checked bit-identical to the
reference's `generate_field` on the whole Nyx field first.

Output: tests/golden/config_golden.json (merged, so --only reruns one case).
"""

from __future__ import annotations

import argparse
import hashlib
import importlib.util
import json
import math
import multiprocessing as mp
import os
import struct
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).parent
OUT = HERE / "config_golden.json"
REF_PKG = Path("/root/reference/pkg/src/sdqz")
LARGE_SLAB_ROWS = 16

_ref = None


def load_ref():
    global _ref
    if _ref is None:
        spec = importlib.util.spec_from_file_location(
            "sdqz_ref", REF_PKG / "__init__.py", submodule_search_locations=[str(REF_PKG)])
        mod = importlib.util.module_from_spec(spec)
        sys.modules["sdqz_ref"] = mod
        spec.loader.exec_module(mod)
        _ref = mod
    return _ref


def sha(b) -> str:
    return hashlib.sha256(b).hexdigest()


def slab_digest(slab_hashes: list[str]) -> str:
    """Digest of an ordered list of per-slab SHA-256 hex digests."""
    return sha("".join(slab_hashes).encode())


CONFIGS = {
    "cesm": dict(profile="smooth", dims=(1800, 3600), eb=1e-4),
    "hurricane": dict(profile="smooth", dims=(100, 500, 500), eb=1e-4),
    "hacc": dict(profile="smooth", dims=(280_953_867,), eb=1e-4),
}
for _p, _tag in (("smooth", "smooth"), ("sparse-near-zero", "sparse")):
    for _eb in (1e-2, 1e-3, 1e-4, 1e-5):
        CONFIGS[f"nyx_{_tag}_{_eb:.0e}"] = dict(profile=_p, dims=(512, 512, 512), eb=_eb)
CONFIGS["nyx_smooth_1e-04_slabwise"] = dict(profile="smooth", dims=(512, 512, 512), eb=1e-4,
                                           slabwise=True, check_against="nyx_smooth_1e-04")
CONFIGS["large"] = dict(profile="smooth", dims=(2048, 2048, 1024), eb=1e-4, slabwise=True)


def section_hashes(blob: bytes) -> dict:
    ref = load_ref()
    h = ref.parse_header(blob)
    p = ref.HEADER_SIZE
    out = {"header": sha(blob[:p])}
    for name, size in (("bitwidths", h.cap), ("outliers", 16 * h.n_outliers),
                       ("chunk_bits", 4 * h.n_chunks), ("payload", h.payload_bytes)):
        out[name] = sha(blob[p:p + size])
        p += size
    return out


def header_fields(blob: bytes) -> dict:
    h = load_ref().parse_header(blob)
    return {"eb_resolved_hex": struct.pack("<d", h.eb_resolved).hex(), "cap": h.cap,
            "chunk_size": h.chunk_size, "unit_width": h.unit_width,
            "n_outliers": h.n_outliers, "n_chunks": h.n_chunks,
            "payload_bytes": h.payload_bytes, "archive_bytes": len(blob)}


# ---------------------------------------------------------------- whole field
def run_whole(name, cfg):
    ref = load_ref()
    t0 = time.time()
    f = ref.generate_field(cfg["profile"], cfg["dims"], seed=1).astype(np.float32)
    tg = time.time() - t0
    blob = ref.compress(f, eb=cfg["eb"], mode="valrel")
    tc = time.time() - t0 - tg
    out = ref.decompress(blob)
    td = time.time() - t0 - tg - tc
    h = ref.parse_header(blob)
    err = float(np.abs(out.astype(np.float64) - f.astype(np.float64)).max())
    rec = {"profile": cfg["profile"], "dims": list(cfg["dims"]), "seed": 1, "mode": "valrel",
           "eb": cfg["eb"], "input_sha256": sha(f.tobytes()), "archive_sha256": sha(blob),
           "sections": section_hashes(blob), "output_sha256": sha(out.tobytes()),
           "max_abs_err": err, "eb_resolved": h.eb_resolved, **header_fields(blob),
           "how": "reference compress/decompress on the whole field",
           "ref_seconds": {"generate": round(tg, 1), "compress": round(tc, 1),
                           "decompress": round(td, 1)}}
    assert err <= h.eb_resolved * (1 + 1e-9) + 1e-6, (name, err)
    return rec


# ---------------------------------------------------------------- slab-wise
def smooth_slab(dims, seed, r0, r1):
    """Reference `_smooth` (synthetic.py:25-35) on rows [r0, r1) of axis 0."""
    ref = load_ref()
    rng = np.random.default_rng(seed)
    axes = ref.synthetic._axes(tuple(dims))
    axes[0] = axes[0][r0:r1]
    shape = (r1 - r0,) + tuple(dims[1:])
    field = np.zeros(shape)
    for _ in range(6):
        amp = rng.uniform(0.5, 1.0)
        phase = rng.uniform(0.0, 2.0 * math.pi)
        arg = phase
        for t in axes:
            arg = arg + rng.uniform(1.0, 4.0) * 2.0 * math.pi * t
        field += amp * np.sin(arg)
    return field


_G = {}


def _slab_stats(args):
    dims, seed, r0, r1 = args
    f = smooth_slab(dims, seed, r0, r1).astype(np.float32)
    return r0, float(f.min()), float(f.max()), bool(np.isfinite(f).all()), sha(f.tobytes())


def _slab_quant(args):
    dims, seed, r0, r1, eb, cap, tmp = args
    ref = load_ref()
    from sdqz_ref.dualquant import _compress_region  # the reference's per-slab worker
    f = smooth_slab(dims, seed, r0, r1).astype(np.float32)
    sd = f.shape
    cfg = ref.QuantConfig.for_rank(eb, len(dims), cap=cap)
    dq = ref.prequantize(f, cfg.eb, sd).shaped
    codes, idx, vals = _compress_region(dq, cfg)
    codes = codes.reshape(-1)
    hist = ref.histogram(codes, cap)
    np.save(os.path.join(tmp, f"codes_{r0}.npy"), codes.astype(np.uint16))
    inner = math.prod(dims[1:])
    return r0, hist, idx.astype(np.int64) + r0 * inner, vals.astype(np.float64)


def _slab_deflate(args):
    r0, bw, chunk, tmp = args
    ref = load_ref()
    codes = np.load(os.path.join(tmp, f"codes_{r0}.npy")).astype(np.uint32)
    cb, _ = ref.canonize(bw)
    ds = ref.deflate(ref.encode(codes, cb), chunk)
    return r0, ds.chunk_bit_lengths, ds.payload


def _slab_decode(args):
    dims, r0, r1, path, cap, eb, chunk, c0, c1, off0, off1, bw, rec_lo, rec_hi, rec_off = args
    ref = load_ref()
    from sdqz_ref.dualquant import _reconstruct_region
    inner = math.prod(dims[1:])
    with open(path, "rb") as fh:
        hdr = fh.read(ref.HEADER_SIZE + cap)
        h = ref.parse_header(hdr)
        fh.seek(rec_off + 16 * rec_lo)
        rec = np.frombuffer(fh.read(16 * (rec_hi - rec_lo)),
                            dtype=[("index", "<u8"), ("value", "<f8")])
        bits_off = ref.HEADER_SIZE + cap + 16 * h.n_outliers
        fh.seek(bits_off + 4 * c0)
        bits = np.frombuffer(fh.read(4 * (c1 - c0)), "<u4")
        fh.seek(bits_off + 4 * h.n_chunks + off0)
        payload = fh.read(off1 - off0)
    _, rb = ref.canonize(bw)
    n = (r1 - r0) * inner
    codes = ref.inflate(ref.DeflatedStream(chunk, bits, payload), rb, n)
    cfg = ref.QuantConfig(eb=h.eb_resolved, cap=cap, block_shape=h.block_shape[:h.ndims])
    sd = (r1 - r0,) + tuple(dims[1:])
    idx = rec["index"].astype(np.int64) - r0 * inner
    dq = _reconstruct_region(codes.reshape(sd), idx, rec["value"].astype(np.float64), cfg)
    out = (dq.reshape(-1) * (2.0 * cfg.eb)).astype(np.float32)
    # error-bound check against the regenerated slab
    f = smooth_slab(dims, 1, r0, r1).astype(np.float32).reshape(-1)
    err = float(np.abs(out.astype(np.float64) - f.astype(np.float64)).max())
    return r0, sha(out.tobytes()), err


def run_slabwise(name, cfg, procs):
    """The reference's row-slab decomposition over chunk-aligned slabs (module doc)."""
    ref = load_ref()
    dims, eb, seed, cap = tuple(cfg["dims"]), cfg["eb"], 1, 1024
    inner, n = math.prod(dims[1:]), math.prod(dims)
    chunk = ref.default_chunk_size(n)
    rows = LARGE_SLAB_ROWS
    assert (rows * inner) % chunk == 0 and dims[0] % rows == 0
    slabs = [(r, r + rows) for r in range(0, dims[0], rows)]
    t0 = time.time()
    tmp = tempfile.mkdtemp(prefix=f"sdqz_{name}_", dir="/tmp")
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        st = sorted(pool.map(_slab_stats, [(dims, seed, a, b) for a, b in slabs]))
        vmin = min(s[1] for s in st)
        vmax = max(s[2] for s in st)
        assert all(s[3] for s in st)
        in_hashes = [s[4] for s in st]
        fd = ref.FieldDescriptor(dims, n, vmin, vmax, False, np.dtype(np.float32))
        spec = ref.ErrorBoundSpec("valrel", eb)
        ebr = ref.resolve_error_bound(spec, fd)
        qcfg = ref.QuantConfig.for_rank(ebr, len(dims), cap=cap)
        tq = time.time()
        qs = sorted(pool.map(_slab_quant, [(dims, seed, a, b, ebr, cap, tmp) for a, b in slabs],
                             chunksize=1), key=lambda x: x[0])
        hist = np.sum([q[1] for q in qs], axis=0)
        idx = np.concatenate([q[2] for q in qs]).astype(np.uint64)
        vals = np.concatenate([q[3] for q in qs])
        del qs
        bw = ref.build_tree(hist)
        defl = sorted(pool.map(_slab_deflate, [(a, bw, chunk, tmp) for a, _ in slabs], chunksize=1),
                      key=lambda x: x[0])
        bits = np.concatenate([d[1] for d in defl]).astype(np.uint32)
        payload = b"".join(d[2] for d in defl)
        del defl
        tc = time.time() - tq
        # the reference's serialize (archive.py:96-137) with a stand-in code array of
        # the right length (serialize reads only qout.codes.size, dims and outliers)
        qout = ref.QuantOutput(np.broadcast_to(np.uint32(0), (n,)), idx, vals, dims, qcfg)
        blob = ref.serialize(qout, ref.DeflatedStream(chunk, bits, payload), bw, qcfg, spec,
                             np.float32)
        path = os.path.join(tmp, "archive.sdqz")
        with open(path, "wb") as fh:
            fh.write(blob)
        h = ref.parse_header(blob)
        # decompress: each slab's chunk range and outlier sub-range (dualquant.py:322-329)
        offs = np.zeros(h.n_chunks + 1, np.int64)
        np.cumsum((bits.astype(np.int64) + 7) >> 3, out=offs[1:])
        rec_off = ref.HEADER_SIZE + cap
        jobs = []
        for a, b in slabs:
            lo, hi = a * inner, b * inner
            c0, c1 = lo // chunk, hi // chunk
            ra, rb_ = (int(x) for x in np.searchsorted(idx, (lo, hi)))
            jobs.append((dims, a, b, path, cap, eb, chunk, c0, c1, int(offs[c0]), int(offs[c1]),
                         bw, ra, rb_, rec_off))
        td0 = time.time()
        dec = sorted(pool.map(_slab_decode, jobs, chunksize=1))
        td = time.time() - td0
    err = max(d[2] for d in dec)
    assert err <= h.eb_resolved * (1 + 1e-9) + 1e-6, err
    for f_ in os.listdir(tmp):
        os.remove(os.path.join(tmp, f_))
    os.rmdir(tmp)
    return {"profile": cfg["profile"], "dims": list(dims), "seed": seed, "mode": "valrel",
            "eb": eb, "slab_rows": rows,
            "input_slab_digest": slab_digest(in_hashes), "archive_sha256": sha(blob),
            "sections": section_hashes(blob), "output_slab_digest": slab_digest([d[1] for d in dec]),
            "max_abs_err": err, "eb_resolved": h.eb_resolved, **header_fields(blob),
            "how": ("reference row-slab decomposition (the workers>1 path of compress_field / "
                    "reconstruct_field) over chunk-aligned slabs, stage functions of the reference"),
            "ref_seconds": {"total": round(time.time() - t0, 1), "compress": round(tc, 1),
                            "decompress": round(td, 1)}, "procs": procs}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--procs", type=int, default=7)
    a = ap.parse_args()
    load_ref()
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    names = a.only or list(CONFIGS)
    # the slab generator must reproduce the reference's generate_field bit for bit
    ref = load_ref()
    for dims in ((64, 48, 40), (33, 17, 29), (1000, 777), (123457,)):
        whole = ref.generate_field("smooth", dims, seed=1)
        cut = [0, 7, dims[0] // 2, dims[0]]
        parts = [smooth_slab(dims, 1, cut[i], cut[i + 1]) for i in range(3)]
        assert np.array_equal(np.concatenate(parts).view(np.uint64), whole.view(np.uint64)), dims
    for name in names:
        cfg = CONFIGS[name]
        t0 = time.time()
        rec = run_slabwise(name, cfg, a.procs) if cfg.get("slabwise") else run_whole(name, cfg)
        if cfg.get("check_against"):
            other = data.get(cfg["check_against"])
            assert other is not None, "run the whole-field case first"
            assert rec["archive_sha256"] == other["archive_sha256"], "slab recipe != whole field"
            rec["matches_whole_field"] = cfg["check_against"]
        data[name] = rec
        OUT.write_text(json.dumps(data, indent=1, sort_keys=True))
        print(f"{name}: {rec['archive_bytes']} B sha {rec['archive_sha256'][:16]} "
              f"({time.time() - t0:.0f} s)", flush=True)


if __name__ == "__main__":
    main()
