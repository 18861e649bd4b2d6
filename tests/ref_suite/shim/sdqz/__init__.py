"""`sdqz` -> the B200 drop-in (paper_2007_09625_b200), so the reference's own
test suite (synced into tests/ref_suite/_ref by tools/sync_ref_suite.py) runs
unmodified against the GPU path.  Test infrastructure only."""

import importlib
import sys

import paper_2007_09625_b200 as _pkg
from paper_2007_09625_b200 import *  # noqa: F401,F403
from paper_2007_09625_b200 import __all__  # noqa: F401

__version__ = getattr(_pkg, "__version__", "0.1.0")
for _m in ("archive", "core", "dualquant", "huffman", "metrics", "pipeline", "synthetic", "cli"):
    sys.modules[f"{__name__}.{_m}"] = importlib.import_module(f"paper_2007_09625_b200.{_m}")
