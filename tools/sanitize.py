"""Small-shape workload touching every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize.py

fast 1D/2D/3D dual-quant and reconstruct (TMA 3D, vectorised 1D/2D), generic
block shapes (strip / row / thread-per-block kernels), f64 input, 64-bit codewords, the warp-parallel decoder and its
sequential hand-back (a corrupted payload), the stage API, the sharded phases
on one rank, quality.  Every result is checked against the oracle."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2007_09625_b200 as S  # noqa: E402
from oracle import sdqz_oracle as O  # noqa: E402


def rt(data, **kw):
    blob = S.compress(data, **kw)
    assert blob == O.compress(data, **kw), kw
    out = S.decompress(blob)
    ref = O.decompress(blob)
    assert np.array_equal(out.view(np.uint8), ref.view(np.uint8))
    return blob


def main():
    rng = np.random.default_rng(7)
    f3 = S.generate_field("smooth", (24, 40, 64), seed=1).astype(np.float32)
    rt(f3, eb=1e-4, mode="valrel")                                  # dq3d_tma, rq3d_block
    rt(S.generate_field("smooth", (40, 256), seed=2).astype(np.float32), eb=1e-4, mode="valrel")  # 2D vec
    rt(S.generate_field("smooth", (5000,), seed=3).astype(np.float32), eb=1e-4, mode="valrel")    # 1D vec
    rt(rng.normal(0, 1, (9, 7, 5)).astype(np.float32), eb=0.02, cap=64, block_shape=(4, 3, 2))     # generic
    rt(S.generate_field("smooth", (20, 33, 40), seed=8).astype(np.float32), eb=1e-4, mode="valrel",
       block_shape=(16, 16, 16))                                     # dq_strip / rq_rows, partial blocks
    rt(S.generate_field("smooth", (7, 11, 90), seed=12).astype(np.float32), eb=1e-4, mode="valrel",
       block_shape=(2, 3, 40))                                       # strip in two lane segments
    rt(S.generate_field("smooth", (60, 100), seed=13).astype(np.float32) + np.float32(3e4), eb=1e-6,
       mode="valrel", block_shape=(16, 30))                          # strip fp64 prediction, idle lanes
    rt(S.generate_field("smooth", (9, 10, 11), seed=14).astype(np.float32), eb=1e-4, mode="valrel",
       block_shape=(4, 4, 4))                                        # dq/rq_blocks (small blocks)
    rt(S.generate_field("smooth", (50, 70), seed=9).astype(np.float32), eb=1e-3, mode="valrel", block_shape=(8, 8))
    rt(rng.normal(0, 1, (12, 12, 12)) * 1e6, eb=1e-3, block_shape=(6, 6, 6))                     # int32 guard: fp64 replay
    rt(S.generate_field("smooth", (20_001,), seed=10).astype(np.float32), eb=1e-4, mode="valrel",
       block_shape=(64,))                                            # dq_rows (1D), rq1d_seg
    rt(S.generate_field("smooth", (200, 300), seed=11).astype(np.float32), eb=1e-4, mode="valrel",
       block_shape=(2, 2))                                           # dq_blocks (many small blocks)
    rt(rng.normal(0, 1, (10, 11, 12)), eb=1e-3, mode="valrel")                                     # f64
    rt(rng.normal(0, 1000, (33, 47)).astype(np.float32), eb=0.01, cap=16)                         # outliers
    fib = [1, 1]
    while len(fib) < 27:
        fib.append(fib[-1] + fib[-2])
    res = np.repeat(np.arange(-13, 14), fib)
    rng.shuffle(res)
    walk = np.cumsum(res).astype(np.float32)
    rt(walk, eb=0.5, cap=64, block_shape=(walk.size,))                                           # 64-bit units
    rt(rng.normal(0, 1, (300,)).astype(np.float32), eb=0.05, chunk_size=7)                       # odd chunks
    # chunks of 65536 codes: the warp decoder's multi-round path (staged rounds, prefetch)
    rt(S.generate_field("smooth", (150000,), seed=4).astype(np.float32), eb=1e-4, mode="valrel", chunk_size=65536)
    rt(S.generate_field("sparse-near-zero", (64, 48, 40), seed=5).astype(np.float32), eb=1e-5, mode="valrel", chunk_size=16384)
    # corrupted payload: the warp decoder hands chunks back to the exact decoder
    blob = bytearray(S.compress(f3, eb=1e-4, mode="valrel"))
    h = S.parse_header(bytes(blob))
    blob[len(blob) - h.payload_bytes + 100] ^= 0x10
    try:
        S.decompress(bytes(blob))
    except (S.CorruptionError, S.SdqzError):
        pass
    # stage API
    cfg = S.QuantConfig(1e-3, 1024, (8, 8, 8))
    q = S.compress_field(f3, S.describe_field(f3, f3.shape), cfg)
    bw = S.build_tree(S.histogram(q.codes, 1024))
    cb, rb = S.canonize(bw)
    ds = S.deflate(S.encode(q.codes, cb), 512)
    assert np.array_equal(S.inflate(ds, rb, q.codes.size), q.codes)
    S.reconstruct_field(q)
    # quality
    S.quality(f3, S.decompress(S.compress(f3, eb=1e-3)))
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
