"""Pin the CPU oracle (oracle/sdqz_oracle.py) against the reference's golden
vectors before it is trusted as the parity checker for the CUDA path."""

import hashlib

import numpy as np
import pytest

from oracle import sdqz_oracle as O

GOLDEN_SHA256 = "ed94702bffa73575db162fb8316d6aff73f0490fd142a29e24b8551929d1ac9a"


def test_golden_archive_sha(golden):
    # recipe of the reference's acceptance criterion 10 (test_acceptance.py:221-227)
    data = (np.random.default_rng(20240117).random((32, 32)) * 4.0 - 2.0).astype(np.float32)
    blob = O.compress(data, eb=1e-3, mode="abs", cap=1024, chunk_size=64)
    assert len(blob) == 12489
    assert hashlib.sha256(blob).hexdigest() == GOLDEN_SHA256
    from conftest import GOLDEN
    assert blob == (GOLDEN / "golden_32x32.sdqz").read_bytes()


def test_archives_bit_exact(golden):
    for e, c in golden.cases():
        blob = O.compress(c["data"], **e["kwargs"])
        assert blob == c["blob"].tobytes(), e["name"]


def test_decompress_bit_exact(golden):
    for e, c in golden.cases():
        out = O.decompress(c["blob"].tobytes())
        assert out.dtype == c["out"].dtype, e["name"]
        assert np.array_equal(out.view(np.uint8), c["out"].view(np.uint8)), e["name"]


def test_stage_vectors(golden):
    for e, c in golden.cases():
        p = O.unpack_archive(c["blob"].tobytes())
        codes, oi, ov = O.dualquant(c["data"], c["data"].shape, p.eb_resolved, p.cap, p.block)
        assert np.array_equal(codes, c["codes"]), e["name"]
        assert np.array_equal(oi, c["oidx"]), e["name"]
        assert np.array_equal(ov.view(np.uint64), c["oval"].view(np.uint64)), e["name"]
        h = O.histogram(codes, p.cap)
        assert np.array_equal(h, c["hist"]), e["name"]
        bw = O.tree_bitwidths(h)
        assert np.array_equal(bw, c["bw"]), e["name"]
        book = O.canonical_book(bw)
        assert book.entries.dtype == c["entries"].dtype
        assert np.array_equal(book.entries, c["entries"]), e["name"]


def test_tree_vectors(golden):
    g = golden.npz
    lens, freq, bw = g["tree_lens"], g["tree_freq"], g["tree_bw"]
    off = 0
    for n in lens.tolist():
        assert np.array_equal(O.tree_bitwidths(freq[off:off + n]), bw[off:off + n])
        off += n


class TestKats:
    """Known-answer tests from the reference suite (SURVEY.md §4 KAT table)."""

    def test_prequant(self):
        assert O.prequant(np.array([0.74]), 0.25).tolist() == [1.0]
        assert O.prequant(np.array([-0.75, 0.75]), 0.25).tolist() == [-2.0, 2.0]
        assert O.prequant(np.array([-0.3]), 0.1).tolist() == [-1.0]  # division, not recip-mul

    def test_tree(self):
        assert O.tree_bitwidths(np.array([5, 2, 1, 1])).tolist() == [1, 2, 3, 3]
        assert O.tree_bitwidths(np.array([0, 9, 0, 0])).tolist() == [0, 1, 0, 0]
        assert O.tree_bitwidths(np.array([1000, 1])).tolist() == [1, 1]
        with pytest.raises(O.OracleError, match="all-zero"):
            O.tree_bitwidths(np.zeros(8, np.int64))

    def test_canonize(self):
        b = O.canonical_book(np.array([1, 2, 3, 3], np.uint8))
        assert b.unit == 32 and int(b.entries[2]) == 0x03000006
        with pytest.raises(O.OracleError, match="Kraft"):
            O.canonical_book(np.array([1, 2, 3], np.uint8))

    def test_unit_width(self):
        assert [O.unit_width(w) for w in (1, 24, 25, 56)] == [32, 32, 64, 64]
        with pytest.raises(O.OracleError, match="57"):
            O.unit_width(57)

    def test_deflate(self):
        units = np.array([(3 << 24) | 0b110, (2 << 24) | 0b01], np.uint32)
        bits, pay = O.deflate(units, 16)
        assert bits.tolist() == [5] and pay == bytes([0b11001000])
        bits, pay = O.deflate(units, 1)
        assert bits.tolist() == [3, 2] and pay == bytes([0b11000000, 0b01000000])

    def test_inflate(self):
        book = O.canonical_book(O.tree_bitwidths(np.array([5, 2, 1, 1])))
        assert O.inflate(np.array([5], np.uint32), bytes([0b11010000]), 8, book, 2).tolist() == [2, 1]
        with pytest.raises(O.OracleCorruption, match="disagree"):
            O.inflate(np.array([5], np.uint32), bytes([0b11001000]), 8, book, 2)

    def test_chunk_size(self):
        assert [O.default_chunk_size(n) for n in (1, 262144, 10**7, 10**10)] == [256, 256, 512, 65536]

    def test_dualquant_kats(self):
        # the reference KATs feed prequantized units (test_dualquant.py:76-96): d = 2*eb*units
        codes, oi, _ = O.dualquant(np.full((2, 2), 6.0), (2, 2), 1.0, 16, (2, 2))
        assert codes.tolist() == [11, 8, 8, 8] and oi.size == 0
        codes, oi, ov = O.dualquant(np.array([16.0]), (1,), 1.0, 16, (1,))
        assert codes.tolist() == [0] and ov.tolist() == [8.0]
        codes, oi, _ = O.dualquant(np.array([-14.0]), (1,), 1.0, 16, (1,))
        assert codes.tolist() == [1] and oi.size == 0
        codes, oi, ov = O.dualquant(np.array([-16.0]), (1,), 1.0, 16, (1,))
        assert codes.tolist() == [0] and ov.tolist() == [-8.0]
        codes, _, _ = O.dualquant(np.zeros(64), (64,), 0.01, 1024, (32,))
        assert (codes == 512).all()
