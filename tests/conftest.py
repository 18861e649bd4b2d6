"""Test configuration: the `gpu` marker, repo-root imports, fixture loading."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).parent / "golden"
# the reference's own suite runs in a subprocess (tests/test_ref_suite.py)
collect_ignore = ["ref_suite"]

try:
    from hypothesis import settings
    settings.register_profile("suite", deadline=None, max_examples=40)
    settings.load_profile("suite")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


class Golden:
    """Reference-generated vectors (tests/golden/make_golden.py)."""

    def __init__(self):
        self.index = json.loads((GOLDEN / "golden_index.json").read_text())
        self.npz = np.load(GOLDEN / "golden.npz")

    def case(self, key):
        g = self.npz
        return {k: g[f"{key}_{k}"] for k in ("data", "blob", "out", "codes", "oidx", "oval",
                                             "hist", "bw", "entries", "chunk_bits")}

    def cases(self):
        for e in self.index:
            yield e, self.case(e["key"])


@pytest.fixture(scope="session")
def golden():
    return Golden()
