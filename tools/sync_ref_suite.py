"""Copy the reference's own test suite (/root/reference/pkg/tests, CLI tests
included: paper_2007_09625_b200/cli.py routes the CLI through the GPU) into tests/ref_suite/_ref, a
git-ignored directory that travels to the GPU box with the repo snapshot.
tests/test_ref_suite.py runs it there against the drop-in through the `sdqz`
shim (tests/ref_suite/shim).  The golden archive the reference's acceptance
test reads (data/golden_32x32.sdqz, absent from the mount) is the one the
reference itself produced (tests/golden/make_golden.py)."""
import shutil
import sys
from pathlib import Path

SRC = Path("/root/reference/pkg/tests")
ROOT = Path(__file__).resolve().parents[1]
DST = ROOT / "tests" / "ref_suite" / "_ref"
FILES = ("conftest.py", "reference.py", "test_acceptance.py", "test_archive.py", "test_core.py",
         "test_dualquant.py", "test_huffman.py", "test_metrics.py", "test_cli.py")


def main() -> int:
    if not SRC.is_dir():
        print(f"{SRC} not present; nothing to sync")
        return 0
    (DST / "data").mkdir(parents=True, exist_ok=True)
    for f in FILES:
        shutil.copyfile(SRC / f, DST / f)
    shutil.copyfile(ROOT / "tests" / "golden" / "golden_32x32.sdqz", DST / "data" / "golden_32x32.sdqz")
    print(f"synced {len(FILES)} files into {DST}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
