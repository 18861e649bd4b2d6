"""Kernel variants behind environment switches stay bit-exact: each switch is
read once per process, so every case runs in a fresh interpreter that
compresses / decompresses a few fields through the package and compares
archive bytes and decompressed bits with the oracle (oracle/sdqz_oracle.py).

  SDQZ_DEC_NS=3|6   the u64 three-codeword / u128 six-codeword decode tables
                    (default: by the stream's mean code length)
  SDQZ_NO_TMA=1     3D dual-quant without the TMA tile pipeline
  SDQZ_NO_VEC1D=1   scalar 1D dual-quant / reconstruct
  SDQZ_NO_VEC2D=1   scalar 2D dual-quant / reconstruct
  SDQZ_NO_GRAPH=1   no CUDA-graph replay of the pipelines
  SDQZ_NO_FORK=1    decompress on one stream (no forked outlier-index branch)
  SDQZ_NO_HEADS=1   1D packer re-reads the input for outlier block heads (no dual-quant side channel)
  SDQZ_PACK_RUNS_MIN=256  register-run packer for every chunk size (default: chunks >= 32768)
  SDQZ_DEC_TARGET=24      short decoder slices (many rounds per chunk)
  SDQZ_NO_BLK=1     generic block shapes on the per-point kernels (not thread-per-block)
  SDQZ_DQ_ROWS=0|1  generic-shape dual-quant thread per block / per block-row segment
  SDQZ_STRIP=0|1    2D/3D generic-shape dual-quant warp per strip of block columns off / for every size
  SDQZ_RQ_ROWS=0|1  2D/3D generic-shape reconstruct warp per strip of block columns off / for every size
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2007_09625_b200 as S
from oracle import sdqz_oracle as O

def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)

rng = np.random.default_rng(5)
fields = [
    (S.generate_field("smooth", (24, 40, 56), seed=3).astype(np.float32), dict(eb=1e-4, mode="valrel")),
    (S.generate_field("smooth", (24, 40, 56), seed=4).astype(np.float32), dict(eb=2e-6, mode="valrel")),
    (S.generate_field("smooth", (300, 451), seed=5).astype(np.float32), dict(eb=1e-3, mode="valrel")),
    (np.cumsum(rng.normal(0, 1, 200_003)).astype(np.float32), dict(eb=0.01, mode="abs")),
    (rng.normal(0, 3, (17, 33, 65)).astype(np.float32), dict(eb=0.05, mode="abs", chunk_size=333)),
    (S.generate_field("smooth", (21, 34, 45), seed=6).astype(np.float32),
     dict(eb=1e-4, mode="valrel", block_shape=(4, 4, 4))),
    (S.generate_field("smooth", (90, 77), seed=7).astype(np.float32),
     dict(eb=1e-3, mode="valrel", block_shape=(8, 8))),
    (S.generate_field("smooth", (7, 11, 70), seed=8).astype(np.float32),
     dict(eb=1e-4, mode="valrel", block_shape=(2, 3, 33))),
    (S.generate_field("smooth", (40, 100), seed=9).astype(np.float32),
     dict(eb=0.01, mode="abs", block_shape=(3, 7))),
    (S.generate_field("smooth", (5, 9, 83), seed=10),
     dict(eb=1e-5, mode="valrel", block_shape=(2, 2, 40))),
]
for f, kw in fields:
    blob = S.compress(f, **kw)
    ref = O.compress(f, **kw)
    assert blob == ref, ("archive differs", f.shape, kw)
    assert np.array_equal(bits(S.decompress(blob)), bits(O.decompress(ref))), ("output differs", f.shape, kw)
print("ok", len(fields))
"""


@pytest.mark.gpu
@pytest.mark.parametrize("env", ["SDQZ_DEC_NS=3", "SDQZ_DEC_NS=6", "SDQZ_NO_TMA=1", "SDQZ_NO_VEC1D=1", "SDQZ_NO_VEC2D=1",
                                 "SDQZ_NO_GRAPH=1", "SDQZ_NO_FORK=1", "SDQZ_NO_HEADS=1", "SDQZ_PACK_RUNS_MIN=256",
                                 "SDQZ_DEC_TARGET=24", "SDQZ_NO_BLK=1", "SDQZ_DQ_ROWS=0", "SDQZ_DQ_ROWS=1",
                                 "SDQZ_RQ_ROWS=0", "SDQZ_RQ_ROWS=1", "SDQZ_STRIP=0", "SDQZ_STRIP=1"])
def test_variant_bit_exact(env):
    k, v = env.split("=")
    e = dict(os.environ, **{k: v})
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], env=e, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.strip().startswith("ok"), r.stdout
