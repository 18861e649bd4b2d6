"""CPU checks of the drop-in boundary: libsdqz_cuda.so loads without a GPU and
exports every entry point include/sdqz_cuda.h declares (no compute calls)."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared():
    text = (ROOT / "include" / "sdqz_cuda.h").read_text()
    return sorted(set(re.findall(r"SDQZ_API\s+[\w\s\*]+?\b(sdqz_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    assert "sdqz_compress" in names and "sdqz_decompress" in names and len(names) >= 20


def test_library_exports_every_declared_symbol():
    from paper_2007_09625_b200 import _lib
    lib = _lib.load_library()
    for name in declared():
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTS) == set(declared())


def test_library_is_sm100a():
    import subprocess
    from paper_2007_09625_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_2007_09625_b200 as S
    with pytest.raises(RuntimeError, match="CUDA"):
        S.compress(np.zeros(16, np.float32), eb=0.1)
