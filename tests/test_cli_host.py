"""CLI host paths (no GPU): argument parsing, dims/env validation, gen -- the
reference's own CLI tests run against the GPU path in tests/test_ref_suite.py."""
import numpy as np
import pytest

from paper_2007_09625_b200 import generate_field
from paper_2007_09625_b200.cli import main


def run(capsys, *argv):
    code = main([str(a) for a in argv])
    out = capsys.readouterr()
    return code, out.out, out.err


def test_gen_matches_generate_field(tmp_path, capsys):
    f = tmp_path / "s.f32"
    code, out, _ = run(capsys, "gen", "--profile", "smooth", "--dims", "12x20", "--seed", 4, "-o", f)
    assert code == 0 and out.strip() == "bytes_written=960"
    assert np.array_equal(np.fromfile(f, "<f4"), generate_field("smooth", (12, 20), seed=4).astype("<f4").ravel())


def test_gen_f64_constant(tmp_path, capsys):
    f = tmp_path / "c.f64"
    code, _, _ = run(capsys, "gen", "--profile", "constant", "--dims", "7", "--value", "2.5",
                     "--dtype", "f64", "-o", f)
    assert code == 0 and np.array_equal(np.fromfile(f, "<f8"), np.full(7, 2.5))


@pytest.mark.parametrize("dims,msg", [("8xq", "cannot parse dims"), ("0x4", "positive extents"),
                                      ("2x2x2x2x2", "positive extents")])
def test_bad_dims(tmp_path, capsys, dims, msg):
    code, _, err = run(capsys, "compress", "-i", tmp_path / "x", "--dims", dims, "--eb", 0.1,
                       "-o", tmp_path / "y")
    assert code == 1 and msg in err and err.startswith("error:")


def test_size_mismatch_names_both_counts(tmp_path, capsys):
    raw = tmp_path / "f.f32"
    np.zeros(100, "<f4").tofile(raw)
    code, _, err = run(capsys, "compress", "-i", raw, "--dims", "9x9", "--eb", 0.1, "-o", tmp_path / "a")
    assert code == 1 and "100" in err and "81" in err


def test_bad_threads_env(tmp_path, capsys, monkeypatch):
    raw = tmp_path / "f.f32"
    np.zeros(16, "<f4").tofile(raw)
    monkeypatch.setenv("SDQZ_THREADS", "zero")
    code, _, err = run(capsys, "compress", "-i", raw, "--dims", "16", "--eb", 0.1, "-o", tmp_path / "a")
    assert code == 1 and "SDQZ_THREADS" in err


def test_bad_ebs(tmp_path, capsys):
    raw = tmp_path / "f.f32"
    np.zeros(16, "<f4").tofile(raw)
    code, _, err = run(capsys, "sweep", "-i", raw, "--dims", "16", "--ebs", "a,b")
    assert code == 1 and "--ebs" in err


def test_missing_input_is_an_error(tmp_path, capsys):
    code, _, err = run(capsys, "decompress", "-i", tmp_path / "nope.sdqz", "-o", tmp_path / "o")
    assert code == 1 and err.startswith("error:")
