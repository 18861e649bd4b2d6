"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src/sdqz
under the alias `sdqz_ref` and records, for a corpus of seeded inputs, the
reference's own outputs: whole archives, decompressed fields, and every
stage-level intermediate (codes, outliers, histogram, bitwidths, packed
codebook, chunk bit lengths, payload).  The fixtures travel with the repo;
/root/reference does not, so nothing at test time reads the reference.
"""

from __future__ import annotations

import hashlib
import importlib.util
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).parent
REF_PKG = Path("/root/reference/pkg/src/sdqz")
GOLDEN_SHA256 = "ed94702bffa73575db162fb8316d6aff73f0490fd142a29e24b8551929d1ac9a"


def load_ref():
    spec = importlib.util.spec_from_file_location(
        "sdqz_ref", REF_PKG / "__init__.py", submodule_search_locations=[str(REF_PKG)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["sdqz_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def archive_cases(rng):
    """(name, data, kwargs) covering ranks, block shapes, caps, modes, dtypes,
    chunk sizes, outlier-heavy and degenerate fields."""
    cases = []

    def add(name, data, **kw):
        cases.append((name, data, kw))

    add("golden_32x32", (np.random.default_rng(20240117).random((32, 32)) * 4.0 - 2.0)
        .astype(np.float32), eb=1e-3, mode="abs", cap=1024, chunk_size=64)
    for rank, dims in ((1, (5000,)), (2, (70, 90)), (3, (20, 24, 28))):
        f = rng.normal(0, 1, dims).cumsum(axis=-1).astype(np.float32)
        add(f"walk_r{rank}_valrel", f, eb=1e-3, mode="valrel")
        add(f"walk_r{rank}_abs_cap64", f, eb=0.02, mode="abs", cap=64)
    add("smooth3d_valrel1e-4", None, profile=("smooth", (40, 50, 60), 1), eb=1e-4, mode="valrel")
    add("smooth2d_valrel1e-4", None, profile=("smooth", (180, 360), 1), eb=1e-4, mode="valrel")
    add("smooth1d_valrel1e-4", None, profile=("smooth", (100_000,), 1), eb=1e-4, mode="valrel")
    add("sparse3d_valrel1e-3", None, profile=("sparse-near-zero", (32, 32, 32), 3), eb=1e-3,
        mode="valrel")
    add("smooth3d_valrel1e-3_cap65536", None, profile=("smooth", (48, 48, 48), 5), eb=1e-3,
        mode="valrel", cap=65536)
    add("noise2d_outlier_heavy", rng.normal(0, 1000, (33, 47)).astype(np.float32), eb=0.01,
        cap=16)
    add("odd_blocks_3d", rng.normal(0, 4, (9, 7, 5)).astype(np.float32), eb=0.02, cap=64,
        block_shape=(4, 3, 2))
    add("odd_blocks_2d", rng.normal(0, 2, (33, 17)).astype(np.float32), eb=0.01, cap=128,
        block_shape=(5, 6))
    add("odd_blocks_1d", rng.normal(0, 1, (400,)).astype(np.float32), eb=1e-3, cap=64,
        block_shape=(7,))
    add("f64_input_3d", rng.normal(0, 1, (10, 11, 12)), eb=1e-3, mode="valrel")
    add("constant_abs", np.full((64, 64), 1.234, np.float32), eb=1e-3, mode="abs")
    add("zeros_1d", np.zeros(1024, np.float32), eb=0.01, mode="abs")
    add("single_point", np.array([0.74], np.float32), eb=0.25)
    nz = np.empty(256, np.float32)
    nz[0::2] = rng.integers(3, 9, 128)
    nz[1::2] = -rng.uniform(0.01, 0.49, 128)
    add("negzero_outliers", nz, eb=0.5, cap=4, block_shape=(256,))
    # residual counts follow Fibonacci numbers -> deepest codeword > 24 bits -> 64-bit units
    fib = [1, 1]
    while len(fib) < 27:
        fib.append(fib[-1] + fib[-2])
    res = np.repeat(np.arange(-13, 14), fib)
    rng.shuffle(res)
    walk = np.cumsum(res).astype(np.float32)
    add("fibonacci_u64_1d", walk, eb=0.5, cap=64, block_shape=(walk.size,))
    add("chunk1", rng.normal(0, 1, (300,)).astype(np.float32), eb=0.05, chunk_size=1)
    add("chunk7", rng.normal(0, 1, (20, 30)).astype(np.float32), eb=0.05, chunk_size=7)
    add("cap4", rng.normal(0, 1, (8, 8, 8)).astype(np.float32), eb=0.05, cap=4)
    add("huge_values_abs", (rng.normal(0, 1, (12, 12, 12)) * 1e30).astype(np.float32),
        eb=1e-3, mode="abs")
    add("big_offset_valrel", (1e6 + rng.normal(0, 1, (16, 16, 16))).astype(np.float32),
        eb=1e-6, mode="valrel")
    add("ties_half", (np.arange(-40, 40, dtype=np.float32) * 0.25), eb=0.125)
    return cases


def main():
    ref = load_ref()
    rng = np.random.default_rng(1234)
    arrays = {}
    index = []
    for i, (name, data, kw) in enumerate(archive_cases(rng)):
        prof = kw.pop("profile", None)
        if prof is not None:
            data = ref.generate_field(prof[0], prof[1], seed=prof[2]).astype(np.float32)
        blob = ref.compress(data, **kw)
        out = ref.decompress(blob)
        ar = ref.deserialize(blob)
        h = ar.header
        cfg = ref.QuantConfig(h.eb_resolved, h.cap, h.block_shape[:h.ndims])
        fd = ref.describe_field(data, data.shape)
        q = ref.compress_field(data, fd, cfg)
        freq = ref.histogram(q.codes, h.cap)
        bw = ref.build_tree(freq)
        cb, _ = ref.canonize(bw)
        key = f"c{i:02d}"
        arrays[f"{key}_data"] = data
        arrays[f"{key}_blob"] = np.frombuffer(blob, np.uint8)
        arrays[f"{key}_out"] = out
        arrays[f"{key}_codes"] = q.codes.astype(np.uint32)
        arrays[f"{key}_oidx"] = q.outlier_indices
        arrays[f"{key}_oval"] = q.outlier_values
        arrays[f"{key}_hist"] = freq
        arrays[f"{key}_bw"] = bw
        arrays[f"{key}_entries"] = cb.entries
        arrays[f"{key}_chunk_bits"] = ar.chunk_bit_lengths
        index.append({"key": key, "name": name, "kwargs": kw, "dims": list(data.shape),
                      "dtype": str(data.dtype), "sha256": hashlib.sha256(blob).hexdigest(),
                      "bytes": len(blob), "n_outliers": int(h.n_outliers),
                      "unit": int(h.unit_width), "chunk": int(h.chunk_size)})
        if name == "golden_32x32":
            assert hashlib.sha256(blob).hexdigest() == GOLDEN_SHA256, "golden SHA mismatch"
            (HERE / "golden_32x32.sdqz").write_bytes(blob)
        print(f"{key} {name:28s} {len(blob):8d} B  outliers={h.n_outliers} unit={h.unit_width}")

    # tree / codebook vectors: tie-heavy small alphabets and wide alphabets
    trng = np.random.default_rng(77)
    freqs, bws = [], []
    for t in range(400):
        k = int(trng.integers(1, 40)) if t < 300 else int(trng.integers(64, 1025))
        cap = 1 << int(np.ceil(np.log2(max(k, 4))))
        f = np.zeros(cap, np.int64)
        hi = 4 if t % 2 == 0 else 100000
        f[trng.choice(cap, k, replace=False)] = trng.integers(1, hi, k)
        freqs.append(f)
        bws.append(ref.build_tree(f))
    fib = [1, 1]
    while len(fib) < 30:
        fib.append(fib[-1] + fib[-2])
    f = np.zeros(32, np.int64)
    f[:30] = fib
    freqs.append(f)
    bws.append(ref.build_tree(f))
    lens = np.array([len(f) for f in freqs], np.int64)
    arrays["tree_lens"] = lens
    arrays["tree_freq"] = np.concatenate(freqs)
    arrays["tree_bw"] = np.concatenate(bws)

    np.savez_compressed(HERE / "golden.npz", **arrays)
    (HERE / "golden_index.json").write_text(json.dumps(index, indent=1))
    print("wrote", HERE / "golden.npz")


if __name__ == "__main__":
    main()
