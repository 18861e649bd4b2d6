"""The reference-side ctypes binding shown in INTEGRATION.md §2
(tests/integration_stub.py, verbatim in the document) runs against the built
library: byte-identical archives and bit-identical outputs vs the oracle,
the reference's exception classes and messages."""
import importlib.util
import os
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
STUB = ROOT / "tests" / "integration_stub.py"


def test_stub_is_the_documented_binding():
    doc = (ROOT / "INTEGRATION.md").read_text()
    assert STUB.read_text().strip() in doc


@pytest.mark.gpu
def test_stub_roundtrip():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    os.environ["SDQZ_CUDA_LIB"] = str(ROOT / "paper_2007_09625_b200" / "libsdqz_cuda.so")
    spec = importlib.util.spec_from_file_location("sdqz_gpu_stub", STUB)
    g = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(g)
    import paper_2007_09625_b200 as S
    from oracle import sdqz_oracle as O

    def bits(a):
        return np.ascontiguousarray(a).view(np.uint32 if a.dtype == np.float32 else np.uint64)

    rng = np.random.default_rng(2)
    cases = [(S.generate_field("smooth", (40, 50, 60), seed=1).astype(np.float32), dict(eb=1e-4, mode="valrel")),
             (np.cumsum(rng.normal(0, 1, 50_001)), dict(eb=0.01, mode="abs", chunk_size=777)),
             (S.generate_field("smooth", (120, 130), seed=2).astype(np.float32),
              dict(eb=1e-3, mode="valrel", cap=256, block_shape=(8, 4)))]
    for f, kw in cases:
        blob = g.compress(f, **kw)
        assert blob == O.compress(f, **kw)
        out = g.decompress(blob)
        assert out.shape == f.shape and np.array_equal(bits(out), bits(O.decompress(blob)))
    with pytest.raises(S.SdqzError, match="mode"):
        g.compress(np.zeros(8, np.float32), eb=0.1, mode="pointwise")
    blob = bytearray(g.compress(cases[0][0], eb=1e-4, mode="valrel"))
    blob[:4] = b"XXXX"
    with pytest.raises(S.ArchiveFormatError):
        g.decompress(bytes(blob))
