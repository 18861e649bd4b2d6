"""The reference's own test suite (pkg/tests, CLI included), unmodified,
against the drop-in on the GPU: `sdqz` resolves to paper_2007_09625_b200
through tests/ref_suite/shim (SURVEY.md §4 lists this suite first)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SUITE = ROOT / "tests" / "ref_suite" / "_ref"


@pytest.mark.gpu
def test_reference_suite_passes_on_the_drop_in():
    if not (SUITE / "test_acceptance.py").exists():
        pytest.skip("reference suite not synced (python tools/sync_ref_suite.py, needs /root/reference)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests" / "ref_suite" / "shim"), str(ROOT),
                                         env.get("PYTHONPATH", "")])
    r = subprocess.run([sys.executable, "-m", "pytest", str(SUITE), "-q", "-p", "no:cacheprovider",
                        "-rs"],
                       cwd=SUITE, env=env, capture_output=True, text=True, timeout=3000)
    tail = r.stdout[-4000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and " failed" not in r.stdout, tail
