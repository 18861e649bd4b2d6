"""GPU parity: every stage of the CUDA path against the reference's golden
vectors (tests/golden) and the CPU oracle, bit-exact."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2007_09625_b200 as S  # noqa: E402
from oracle import sdqz_oracle as O  # noqa: E402


def bits(a):
    a = np.asarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


class TestGoldenArchives:
    def test_compress_bytes(self, golden):
        for e, c in golden.cases():
            blob = S.compress(c["data"], **e["kwargs"])
            assert blob == c["blob"].tobytes(), e["name"]

    def test_decompress_bits(self, golden):
        for e, c in golden.cases():
            out = S.decompress(c["blob"].tobytes())
            assert out.dtype == c["out"].dtype and out.shape == c["out"].shape, e["name"]
            assert np.array_equal(bits(out), bits(c["out"])), e["name"]

    def test_device_resident_roundtrip(self, golden):
        for e, c in golden.cases():
            t = torch.from_numpy(np.ascontiguousarray(c["data"])).cuda()
            dev = S.compress_device(t, **e["kwargs"])
            assert dev.to_bytes() == c["blob"].tobytes(), e["name"]
            out = S.decompress_device(dev).cpu().numpy()
            assert np.array_equal(bits(out), bits(c["out"])), e["name"]


class TestGoldenStages:
    def test_compress_field(self, golden):
        for e, c in golden.cases():
            h = S.parse_header(c["blob"].tobytes())
            cfg = S.QuantConfig(h.eb_resolved, h.cap, h.block_shape[:h.ndims])
            fd = S.describe_field(c["data"], c["data"].shape)
            q = S.compress_field(c["data"], fd, cfg)
            assert q.codes.dtype == np.uint32
            assert np.array_equal(q.codes, c["codes"]), e["name"]
            assert np.array_equal(q.outlier_indices, c["oidx"]), e["name"]
            assert np.array_equal(bits(q.outlier_values), bits(c["oval"])), e["name"]

    def test_histogram_tree_canonize(self, golden):
        for e, c in golden.cases():
            cap = int(c["hist"].size)
            h = S.histogram(c["codes"], cap)
            assert h.dtype == np.int64 and np.array_equal(h, c["hist"]), e["name"]
            bw = S.build_tree(h)
            assert np.array_equal(bw, c["bw"]), e["name"]
            cb, rb = S.canonize(bw)
            assert cb.entries.dtype == c["entries"].dtype, e["name"]
            assert np.array_equal(cb.entries, c["entries"]), e["name"]
            ob = O.canonical_book(bw)
            assert np.array_equal(rb.first_codes, ob.first) and np.array_equal(rb.offsets, ob.offsets)
            assert np.array_equal(rb.symbols, ob.symbols) and rb.max_bitwidth == ob.max_bw

    def test_encode_deflate_inflate(self, golden):
        for e, c in golden.cases():
            p = O.unpack_archive(c["blob"].tobytes())
            cb, rb = S.canonize(c["bw"])
            units = S.encode(c["codes"], cb)
            assert np.array_equal(units, O.encode(c["codes"], O.canonical_book(c["bw"])))
            ds = S.deflate(units, p.chunk)
            assert np.array_equal(ds.chunk_bit_lengths, c["chunk_bits"]), e["name"]
            assert ds.payload == p.payload, e["name"]
            got = S.inflate(ds, rb, c["codes"].size)
            assert got.dtype == np.uint32 and np.array_equal(got, c["codes"]), e["name"]

    def test_reconstruct_field(self, golden):
        for e, c in golden.cases():
            h = S.parse_header(c["blob"].tobytes())
            cfg = S.QuantConfig(h.eb_resolved, h.cap, h.block_shape[:h.ndims])
            q = S.QuantOutput(c["codes"], c["oidx"], c["oval"], h.field_dims, cfg)
            got = S.reconstruct_field(q)
            want = O.reconstruct(c["codes"], c["oidx"], c["oval"], h.field_dims, h.eb_resolved,
                                 h.cap, h.block_shape[:h.ndims])
            assert np.array_equal(bits(got), bits(want)), e["name"]

    def test_tree_vectors(self, golden):
        g = golden.npz
        off = 0
        for n in g["tree_lens"].tolist():
            f = g["tree_freq"][off:off + n]
            assert np.array_equal(S.build_tree(f), g["tree_bw"][off:off + n])
            off += n


class TestKats:
    """The reference suite's known answers (SURVEY.md §4 KAT table)."""

    def test_prequantize(self):
        assert S.prequantize(np.array([0.74]), eb=0.25).values[0] == 1.0
        assert S.prequantize(np.array([-0.75, 0.75]), eb=0.25).values.tolist() == [-2.0, 2.0]
        assert S.prequantize(np.array([-0.3]), eb=0.1).values.tolist() == [-1.0]
        with pytest.raises(S.SdqzError, match="nonfinite"):
            S.prequantize(np.array([1.0, np.inf]), eb=0.1)

    def test_postquantize_block(self):
        cfg = S.QuantConfig(eb=1.0, cap=16, block_shape=(2, 2))
        codes, idx, _ = S.postquantize_block(S.pad_block(np.full((2, 2), 3.0)), cfg)
        assert codes.tolist() == [[11, 8], [8, 8]] and idx.size == 0
        cfg1 = S.QuantConfig(eb=1.0, cap=16, block_shape=(1,))
        codes, idx, vals = S.postquantize_block(S.pad_block(np.array([8.0])), cfg1)
        assert codes.tolist() == [0] and vals.tolist() == [8.0]
        codes, idx, _ = S.postquantize_block(S.pad_block(np.array([-7.0])), cfg1)
        assert codes.tolist() == [1] and idx.size == 0

    def test_compress_field_kats(self):
        d = np.zeros(64)
        q = S.compress_field(d, S.describe_field(d, [64]), S.QuantConfig.for_rank(0.01, 1))
        assert np.all(q.codes == 512) and q.n_outliers == 0
        d = np.array([1.0])
        q = S.compress_field(d, S.describe_field(d, [1]), S.QuantConfig.for_rank(0.25, 1))
        assert q.codes.tolist() == [514]

    def test_tree_and_book(self):
        assert S.build_tree(np.array([5, 2, 1, 1])).tolist() == [1, 2, 3, 3]
        assert S.build_tree(np.array([0, 9, 0, 0])).tolist() == [0, 1, 0, 0]
        assert S.build_tree(np.array([1000, 1])).tolist() == [1, 1]
        with pytest.raises(S.SdqzError, match="all-zero"):
            S.build_tree(np.zeros(8, dtype=np.int64))
        cb, rb = S.canonize(np.array([1, 2, 3, 3], dtype=np.uint8))
        assert cb.codewords.tolist() == [0b0, 0b10, 0b110, 0b111]
        assert int(cb.entries[2]) == 0x03000006 and cb.unit_width == 32
        with pytest.raises(S.SdqzError, match="Kraft"):
            S.canonize(np.array([1, 2, 3], dtype=np.uint8))

    def test_deflate_inflate_kats(self):
        units = np.array([(3 << 24) | 0b110, (2 << 24) | 0b01], dtype=np.uint32)
        ds = S.deflate(units, chunk_size=16)
        assert ds.chunk_bit_lengths.tolist() == [5] and ds.payload == bytes([0b11001000])
        ds = S.deflate(units, chunk_size=1)
        assert ds.chunk_bit_lengths.tolist() == [3, 2]
        assert ds.payload == bytes([0b11000000, 0b01000000])
        bw = S.build_tree(np.array([5, 2, 1, 1]))
        cb, rb = S.canonize(bw)
        ds = S.DeflatedStream(8, np.array([5], dtype=np.uint32), bytes([0b11010000]))
        assert S.inflate(ds, rb, 2).tolist() == [2, 1]

    def test_fibonacci_units(self):
        fib = [1, 1]
        while len(fib) < 30:
            fib.append(fib[-1] + fib[-2])
        freq = np.zeros(32, dtype=np.int64)
        freq[:30] = fib
        bw = S.build_tree(freq)
        cb, rb = S.canonize(bw)
        assert int(bw.max()) == 29 and cb.unit_width == 64 and cb.entries.dtype == np.uint64
        codes = np.random.default_rng(5).integers(0, 30, 20_000, dtype=np.uint32)
        ds = S.deflate(S.encode(codes, cb), 256)
        assert np.array_equal(S.inflate(ds, rb, codes.size), codes)


class TestErrors:
    def test_corruption_messages(self):
        bw = S.build_tree(np.array([5, 2, 1, 1]))
        cb, rb = S.canonize(bw)
        bad = S.DeflatedStream(8, np.array([5], dtype=np.uint32), bytes([0b11001000]))
        with pytest.raises(S.CorruptionError, match="disagree"):
            S.inflate(bad, rb, 2)
        cb1, rb1 = S.canonize(S.build_tree(np.array([42, 0, 0, 0])))
        ds = S.deflate(S.encode(np.zeros(100, np.uint32), cb1), 7)
        assert np.array_equal(S.inflate(ds, rb1, 100), np.zeros(100, np.uint32))
        with pytest.raises(S.CorruptionError, match="no codeword"):
            S.inflate(S.DeflatedStream(7, ds.chunk_bit_lengths, b"\xff" + ds.payload[1:]), rb1, 100)
        with pytest.raises(S.CorruptionError, match="outside"):
            S.histogram(np.array([4]), 4)
        _, cbz, _ = (None, *S.canonize(S.build_tree(np.array([5, 0, 3, 2, 0, 0, 0, 0]))))
        with pytest.raises(S.CorruptionError, match="no codebook entry"):
            S.encode(np.array([1]), cbz)

    def test_reconstruct_validation(self):
        d = np.full(8, 5.0)
        cfg = S.QuantConfig.for_rank(0.01, 1)
        q = S.compress_field(d, S.describe_field(d, [8]), cfg)
        q.codes[3] = 0
        with pytest.raises(S.CorruptionError, match="outlier"):
            S.reconstruct_field(q)
        q = S.compress_field(d, S.describe_field(d, [8]), cfg)
        q.outlier_indices = np.array([2], dtype=np.uint64)
        q.outlier_values = np.array([1.0])
        with pytest.raises(S.CorruptionError, match="code is not 0"):
            S.reconstruct_field(q)

    def test_archive_errors_on_device_path(self):
        blob = S.compress(np.linspace(0, 1, 64).reshape(8, 8), eb=0.01)
        with pytest.raises(S.ArchiveFormatError, match="short read"):
            S.decompress(b"")
        b = bytearray(blob)
        b[0] = ord("X")
        with pytest.raises(S.ArchiveFormatError, match="bad magic"):
            S.decompress(bytes(b))
        with pytest.raises(S.ArchiveFormatError, match="trailing"):
            S.decompress(blob + b"\0")
        with pytest.raises(S.ArchiveFormatError, match="short read"):
            S.decompress(blob[:-1])
        h = S.parse_header(blob)
        table = np.frombuffer(blob[S.HEADER_SIZE:S.HEADER_SIZE + h.cap], np.uint8)
        b = bytearray(blob)
        b[S.HEADER_SIZE + int(np.flatnonzero(table)[0])] += 1
        with pytest.raises(S.ArchiveFormatError, match="Kraft"):
            S.decompress(bytes(b))

    def test_compress_errors(self):
        with pytest.raises(S.SdqzError, match="NaN"):
            S.compress(np.array([0.0, np.nan, 1.0], np.float32), eb=0.1)
        with pytest.raises(S.SdqzError, match="NaN"):
            S.compress(np.array([0.0, np.inf, 1.0], np.float32), eb=0.1, mode="valrel")
        with pytest.raises(S.SdqzError, match="absolute"):
            S.compress(np.full(16, 3.0, np.float32), eb=0.1, mode="valrel")
        with pytest.raises(S.SdqzError, match="must be positive"):
            S.compress(np.arange(16, dtype=np.float32), eb=0.0)
        with pytest.raises(S.SdqzError, match="cap"):
            S.compress(np.arange(16, dtype=np.float32), eb=0.1, cap=100)
        with pytest.raises(S.SdqzError, match="NaN"):
            S.compress(np.array([np.nan, 1.0], np.float32), eb=0.1, cap=100)
        with pytest.raises(S.SdqzError, match="mode"):
            S.compress(np.arange(16, dtype=np.float32), eb=0.1, mode="pointwise")


class TestDifferential:
    """Seeded random fields: GPU archive bytes and decompressed bits == oracle."""

    @pytest.mark.parametrize("seed", range(40))
    def test_random_fields(self, seed):
        rng = np.random.default_rng(1000 + seed)
        rank = int(rng.integers(1, 4))
        dims = tuple(int(d) for d in rng.integers(1, [4000, 90, 40][rank - 1], rank))
        kind = seed % 4
        if kind == 0:
            data = rng.normal(0, rng.uniform(0.5, 20), dims)
        elif kind == 1:
            data = np.cumsum(rng.normal(0, 1, dims), axis=-1)
        elif kind == 2:
            data = S.generate_field("smooth", dims, seed=seed)
        else:
            data = rng.normal(0, 1e4, dims)
        data = data.astype(np.float32 if seed % 5 else np.float64)
        cap = int(rng.choice([4, 16, 64, 256, 1024, 4096, 65536]))
        block = None if seed % 3 else tuple(int(b) for b in rng.integers(1, 9, rank))
        mode = "valrel" if seed % 2 else "abs"
        eb = float(rng.uniform(1e-4, 1e-2)) if mode == "valrel" else float(rng.uniform(1e-3, 0.3))
        chunk = None if seed % 4 else int(rng.integers(1, 5000))
        kw = dict(eb=eb, mode=mode, cap=cap, block_shape=block, chunk_size=chunk)
        blob = S.compress(data, **kw)
        ref = O.compress(data, **kw)
        assert blob == ref
        assert np.array_equal(bits(S.decompress(blob)), bits(O.decompress(ref)))


class TestConfigScale:
    """Config-shaped fields at full size: bytes == oracle (Hurricane) and
    size-independent properties for the larger configs."""

    def test_hurricane_bit_exact(self):
        f = S.generate_field("smooth", (100, 500, 500), seed=1).astype(np.float32)
        blob = S.compress(f, eb=1e-4, mode="valrel")
        assert blob == O.compress(f, eb=1e-4, mode="valrel")
        out = S.decompress(blob)
        h = S.parse_header(blob)
        err = np.abs(out.astype(np.float64) - f.astype(np.float64))
        assert err.max() <= h.eb_resolved * (1 + 1e-6) + 2 * np.spacing(np.abs(out).max())

    def test_cesm_roundtrip(self):
        f = S.generate_field("smooth", (1800, 3600), seed=1).astype(np.float32)
        blob = S.compress(f, eb=1e-4, mode="valrel")
        assert blob == O.compress(f, eb=1e-4, mode="valrel")
        out = S.decompress(blob)
        h = S.parse_header(blob)
        assert np.abs(out.astype(np.float64) - f).max() <= h.eb_resolved + 2 * np.spacing(np.float32(8))


class TestCorruptStreams:
    """Bit flips in the payload of medium archives: the warp-parallel decoder
    must hand such chunks to the exact path and raise what the oracle raises
    (or decode identically when the flip still parses)."""

    @pytest.mark.parametrize("seed", range(12))
    def test_payload_bitflips(self, seed):
        rng = np.random.default_rng(seed)
        f = S.generate_field("smooth", (48, 64, 80), seed=seed).astype(np.float32)
        blob = bytearray(S.compress(f, eb=1e-4, mode="valrel"))
        h = S.parse_header(bytes(blob))
        p0 = len(blob) - h.payload_bytes
        for _ in range(int(rng.integers(1, 4))):
            pos = p0 + int(rng.integers(0, h.payload_bytes))
            blob[pos] ^= 1 << int(rng.integers(0, 8))
        blob = bytes(blob)
        try:
            want = O.decompress(blob)
            werr = None
        except O.OracleError as e:
            want, werr = None, e
        if werr is None:
            got = S.decompress(blob)
            assert np.array_equal(bits(got), bits(want))
        else:
            with pytest.raises(S.SdqzError) as ei:
                S.decompress(blob)
            assert str(ei.value) == str(werr)
            assert isinstance(ei.value, S.CorruptionError) == isinstance(werr, O.OracleCorruption)


class TestDualquant3DPaths:
    """The TMA-fed 3D dual-quant kernel (row pitch a multiple of 4 floats):
    partial tasks at every edge, the task redo path (magnitudes at or above
    2^27 units of 2eb, values on prequantization rounding ties), the shared
    and global histogram variants."""

    @staticmethod
    def check(data, **kw):
        blob = S.compress(data, **kw)
        ref = O.compress(data, **kw)
        assert blob == ref
        assert np.array_equal(bits(S.decompress(blob)), bits(O.decompress(ref)))

    @pytest.mark.parametrize("dims", [(8, 8, 32), (13, 17, 36), (9, 8, 64), (3, 5, 4), (17, 9, 100),
                                      (24, 40, 128)])
    def test_edges(self, dims):
        f = S.generate_field("smooth", dims, seed=7).astype(np.float32)
        self.check(f, eb=1e-3, mode="valrel")

    @pytest.mark.parametrize("cap", [4, 16, 32, 1024, 65536])
    def test_caps(self, cap):
        rng = np.random.default_rng(cap)
        f = np.cumsum(rng.normal(0, 1, (12, 20, 40)), axis=-1).astype(np.float32)
        self.check(f, eb=0.05, mode="abs", cap=cap)

    def test_big_magnitudes_redo(self):
        rng = np.random.default_rng(11)
        f = rng.normal(0, 1.0, (16, 24, 64)).astype(np.float32)
        f[3:5, 2:9, 10:50] *= 3e8            # |x / 2eb| well above 2^27 in some tasks
        f[12, 20, 63] = 2.0 ** 27 * 2e-3     # one value right at the int32 bound
        self.check(f, eb=1e-3, mode="abs")

    def test_rounding_ties(self):
        rng = np.random.default_rng(5)
        two_eb = 0.25
        k = rng.integers(-4000, 4000, (16, 16, 32)).astype(np.float64)
        f = ((k + 0.5) * two_eb).astype(np.float32)          # exact ties
        f[::2] = np.nextafter(f[::2], np.float32(np.inf))    # one ulp off the tie
        f[1::4] = np.nextafter(f[1::4], np.float32(-np.inf))
        self.check(f, eb=two_eb / 2, mode="abs")
        g = (k * 0.3 + 0.15).astype(np.float32)               # near-ties for a non-dyadic bound
        self.check(g, eb=0.15, mode="abs")

    def test_nonfinite_abs_mode(self):
        f = np.zeros((8, 8, 32), np.float32)
        f[4, 4, 17] = np.inf
        with pytest.raises(S.SdqzError, match="NaN"):
            S.compress(f, eb=0.1, mode="abs")
        f[4, 4, 17] = np.nan
        with pytest.raises(S.SdqzError, match="NaN"):
            S.compress(f, eb=0.1, mode="abs")


class TestVec1DPaths:
    """The vectorised 1D kernels (dq1d_vec / rq1d_vec: whole 1024-point tasks,
    tail by the scalar kernels): tails, caps, the fp64 task redo, rounding
    ties, outlier values beyond the int32 reset-scan range."""

    check = staticmethod(TestDualquant3DPaths.check)

    @pytest.mark.parametrize("n", [1024, 1025, 2047, 5000, 100_003, 3_000_000])
    def test_lengths(self, n):
        f = S.generate_field("smooth", (n,), seed=3).astype(np.float32)
        self.check(f, eb=1e-4, mode="valrel")

    @pytest.mark.parametrize("cap", [4, 16, 32, 1024, 65536])
    def test_caps(self, cap):
        rng = np.random.default_rng(cap)
        f = np.cumsum(rng.normal(0, 1, 9000)).astype(np.float32)
        self.check(f, eb=0.05, mode="abs", cap=cap)

    def test_big_magnitudes_redo(self):
        rng = np.random.default_rng(12)
        f = rng.normal(0, 1.0, 8192).astype(np.float32)
        f[1500:1700] *= 3e8                  # fp64 task redo in dq, int64 rows in rq
        f[5000] = 2.0 ** 27 * 2e-3           # right at the int32 bound
        f[6000:6040] = 2.0 ** 31 * 2e-3      # outlier values beyond 2^30 units
        self.check(f, eb=1e-3, mode="abs")

    def test_outlier_dense(self):
        rng = np.random.default_rng(13)
        f = rng.normal(0, 50.0, 20000).astype(np.float32)    # most points are outliers
        self.check(f, eb=0.01, mode="abs", cap=16)

    def test_rounding_ties(self):
        rng = np.random.default_rng(6)
        k = rng.integers(-4000, 4000, 4096).astype(np.float64)
        f = ((k + 0.5) * 0.25).astype(np.float32)
        f[::2] = np.nextafter(f[::2], np.float32(np.inf))
        self.check(f, eb=0.125, mode="abs")
        g = (k * 0.3 + 0.15).astype(np.float32)
        self.check(g, eb=0.15, mode="abs")

    def test_nonfinite(self):
        f = np.zeros(4096, np.float32)
        f[3000] = np.nan
        with pytest.raises(S.SdqzError, match="NaN"):
            S.compress(f, eb=0.1, mode="abs")

    def test_float64_output_path(self):
        f = S.generate_field("smooth", (10_000,), seed=4)   # f64 in / out: scalar dq, vec rq
        self.check(f, eb=1e-4, mode="valrel")


class TestRecords1D:
    """1D decompress takes outlier values straight from the archive records
    (rank among a task's zero codes): edited records must raise what the
    oracle raises, or decode identically (non-integer values: fp64 path)."""

    @staticmethod
    def archive():
        rng = np.random.default_rng(21)
        f = np.cumsum(rng.normal(0, 1, 50_000)).astype(np.float32)
        f[::97] += 40.0                      # regular outliers
        blob = S.compress(f, eb=0.05, mode="abs", cap=64)
        h = S.parse_header(blob)
        off = S.HEADER_SIZE + h.cap
        return bytearray(blob), h, off

    @staticmethod
    def outcome(blob):
        try:
            return O.decompress(bytes(blob)), None
        except O.OracleError as e:
            return None, e

    def check(self, blob):
        want, werr = self.outcome(blob)
        if werr is None:
            assert np.array_equal(bits(S.decompress(bytes(blob))), bits(want))
        else:
            with pytest.raises(S.SdqzError) as ei:
                S.decompress(bytes(blob))
            assert str(ei.value) == str(werr)

    def test_roundtrip(self):
        blob, h, off = self.archive()
        assert h.n_outliers > 100
        self.check(blob)

    @pytest.mark.parametrize("edit", ["shift", "swap", "range", "fraction", "huge", "drop_last"])
    def test_edited_records(self, edit):
        blob, h, off = self.archive()
        rec = np.frombuffer(bytes(blob[off:off + 16 * h.n_outliers]), np.uint64).reshape(-1, 2).copy()
        j = h.n_outliers // 2
        if edit == "shift":
            rec[j, 0] += 1
        elif edit == "swap":
            rec[[j, j + 1], 0] = rec[[j + 1, j], 0]
        elif edit == "range":
            rec[-1, 0] = 10 ** 9
        elif edit == "fraction":
            v = np.array([rec[j, 1]], np.uint64).view(np.float64)[0] + 0.25
            rec[j, 1] = np.array([v]).view(np.uint64)[0]
        elif edit == "huge":
            rec[j, 1] = np.array([3.0 * 2 ** 31]).view(np.uint64)[0]
        elif edit == "drop_last":
            rec[-1, 0] += 1
        blob[off:off + 16 * h.n_outliers] = rec.tobytes()
        self.check(blob)


class TestVec2DPaths:
    """The vectorised 2D kernels (dq2d_vec / rq2d_vec: 16 x 128 tasks, rows a
    multiple of 4 floats): edges, caps, the fp64 task redo, rounding ties,
    outliers beyond the int32 range, fp64 fields."""

    check = staticmethod(TestDualquant3DPaths.check)

    @pytest.mark.parametrize("dims", [(16, 128), (17, 132), (1, 4), (40, 300), (123, 1028), (1800, 3600)])
    def test_shapes(self, dims):
        f = S.generate_field("smooth", dims, seed=9).astype(np.float32)
        self.check(f, eb=1e-4, mode="valrel")

    @pytest.mark.parametrize("cap", [4, 16, 32, 1024, 65536])
    def test_caps(self, cap):
        rng = np.random.default_rng(cap + 1)
        f = np.cumsum(rng.normal(0, 1, (40, 200)), axis=1).astype(np.float32)
        self.check(f, eb=0.05, mode="abs", cap=cap)

    def test_big_magnitudes(self):
        rng = np.random.default_rng(14)
        f = rng.normal(0, 1.0, (48, 256)).astype(np.float32)
        f[5:9, 10:90] *= 3e8                 # fp64 task redo in dq, int64 rows in rq
        f[30, 200] = 2.0 ** 27 * 2e-3
        f[40:42, 100:140] = 2.0 ** 30 * 2e-3   # outlier values beyond 2^29 units
        self.check(f, eb=1e-3, mode="abs")

    def test_outlier_dense(self):
        rng = np.random.default_rng(15)
        f = rng.normal(0, 50.0, (64, 320)).astype(np.float32)
        self.check(f, eb=0.01, mode="abs", cap=16)

    def test_rounding_ties(self):
        rng = np.random.default_rng(16)
        k = rng.integers(-4000, 4000, (32, 256)).astype(np.float64)
        f = ((k + 0.5) * 0.25).astype(np.float32)
        f[:, ::2] = np.nextafter(f[:, ::2], np.float32(np.inf))
        self.check(f, eb=0.125, mode="abs")
        g = (k * 0.3 + 0.15).astype(np.float32)
        self.check(g, eb=0.15, mode="abs")

    def test_nonfinite(self):
        f = np.zeros((32, 128), np.float32)
        f[20, 77] = np.inf
        with pytest.raises(S.SdqzError, match="NaN"):
            S.compress(f, eb=0.1, mode="abs")

    def test_float64_field(self):
        f = S.generate_field("smooth", (50, 400), seed=5)
        self.check(f, eb=1e-4, mode="valrel")

    def test_fraction_outlier_block(self):
        # a non-integer outlier value sends its block to the fp64 replay
        rng = np.random.default_rng(17)
        f = np.cumsum(rng.normal(0, 1, (32, 256)), axis=1).astype(np.float32)
        f[::7, ::11] += 30.0
        blob = bytearray(S.compress(f, eb=0.05, mode="abs", cap=64))
        h = S.parse_header(bytes(blob))
        off = S.HEADER_SIZE + h.cap
        rec = np.frombuffer(bytes(blob[off:off + 16 * h.n_outliers]), np.uint64).reshape(-1, 2).copy()
        v = rec[:, 1].copy().view(np.float64)
        v[h.n_outliers // 2] += 0.25
        rec[:, 1] = v.view(np.uint64)
        blob[off:off + 16 * h.n_outliers] = rec.tobytes()
        assert np.array_equal(bits(S.decompress(bytes(blob))), bits(O.decompress(bytes(blob))))


class TestQualityKernel:
    """metrics.quality through sdqz_quality (reference test_metrics.py:10-60)."""

    @staticmethod
    def numpy_quality(a, b):
        a = np.asarray(a, np.float64).ravel()
        b = np.asarray(b, np.float64).ravel()
        d = a - b
        return float(np.sqrt(np.mean(d * d))), float(np.abs(d).max()), float(a.max() - a.min())

    def test_psnr_formula(self):
        orig = np.array([0.0, 1.0])
        q = S.quality(orig, orig + 1e-4)
        assert q.psnr_db == pytest.approx(80.0, abs=1e-9)
        assert q.rmse == pytest.approx(1e-4) and q.max_abs_error == pytest.approx(1e-4)

    def test_identical(self):
        q = S.quality(np.arange(5.0), np.arange(5.0))
        assert q.rmse == 0.0 and np.isinf(q.psnr_db)

    @pytest.mark.parametrize("dt", [np.float32, np.float64])
    def test_against_numpy(self, dt):
        rng = np.random.default_rng(3)
        a = rng.normal(0, 3, 1_234_567).astype(dt)
        b = (a + rng.uniform(-1e-3, 1e-3, a.size)).astype(np.float32)
        q = S.quality(a, b)
        rmse, mx, rg = self.numpy_quality(a, b)
        assert q.max_abs_error == mx and q.value_range == rg
        assert q.rmse == pytest.approx(rmse, rel=1e-12)

    def test_errors(self):
        with pytest.raises(S.SdqzError, match="length"):
            S.quality(np.zeros(3), np.zeros(4))
        with pytest.raises(S.SdqzError, match="zero value range"):
            S.quality(np.zeros(4), np.ones(4))
        with pytest.raises(S.SdqzError, match="nonfinite"):
            S.quality(np.array([0.0, np.nan]), np.zeros(2))

    def test_rd_sweep_matches_decompress(self):
        f = S.generate_field("smooth", (24, 40, 56), seed=2).astype(np.float32)
        fd = S.describe_field(f, f.shape)
        rows = S.rd_sweep(f, fd, [S.ErrorBoundSpec("valrel", e) for e in (1e-2, 1e-3, 1e-4)])
        for r, e in zip(rows, (1e-2, 1e-3, 1e-4)):
            blob = O.compress(f, eb=e, mode="valrel")
            rec = O.decompress(blob)
            rmse, mx, rg = self.numpy_quality(f, rec)
            assert r.error is None and r.max_abs_err == mx
            assert r.psnr_db == pytest.approx(20 * np.log10(rg / rmse), abs=1e-9)
            assert r.cr == pytest.approx(f.nbytes / len(blob))


class TestLargeChunks:
    """Chunks larger than the decoder's shared staging buffer (~4 KB) are read
    from global memory (GlobalReader4): HACC- and large-config-sized chunks."""

    @pytest.mark.parametrize("chunk", [16384, 65536])
    def test_big_chunks(self, chunk):
        rng = np.random.default_rng(chunk)
        f = np.cumsum(rng.normal(0, 1, 400_000)).astype(np.float32)
        kw = dict(eb=0.02, mode="abs", chunk_size=chunk)
        blob = S.compress(f, **kw)
        assert blob == O.compress(f, **kw)
        h = S.parse_header(blob)
        assert h.payload_bytes / h.n_chunks > 8192
        assert np.array_equal(bits(S.decompress(blob)), bits(O.decompress(blob)))

    @pytest.mark.parametrize("eb,chunk", [(3e-2, 32768), (1e-3, 40001), (2e-5, 65536), (1e-6, 32768)])
    def test_register_run_packer(self, eb, chunk):
        """Chunks >= 32768 codes take the register-run packer (chunk_pack32_runs_kernel):
        low to high code entropy (16-, 8- and 4-code sub-runs, runs over 64 bits),
        an odd chunk size (unaligned chunk starts), outliers."""
        f = S.generate_field("smooth", (40, 96, 128), seed=7).astype(np.float32)
        f[::7, ::5, ::3] += np.float32(3.0)
        kw = dict(eb=eb, mode="valrel", chunk_size=chunk)
        blob = S.compress(f, **kw)
        assert blob == O.compress(f, **kw)
        assert np.array_equal(bits(S.decompress(blob)), bits(O.decompress(blob)))

    def test_fused_pack_64bit_units(self):
        """Chunks >= 32768 codes with codewords over 24 bits: the fused 32-bit
        stats + pack kernel stands down and the 64-bit path (stats, scan, run
        packer) packs, decided on the device."""
        rng = np.random.default_rng(11)
        fib = [1, 1]
        while len(fib) < 27:
            fib.append(fib[-1] + fib[-2])
        res = np.repeat(np.arange(-13, 14), fib)
        rng.shuffle(res)
        walk = np.cumsum(np.concatenate([res, res[: 70_000 - res.size]]) if res.size < 70_000 else res)
        walk = walk.astype(np.float32)
        for chunk in (32768, 65536):
            kw = dict(eb=0.5, cap=64, block_shape=(walk.size,), chunk_size=chunk)
            blob = S.compress(walk, **kw)
            assert S.parse_header(blob).unit_width == 64
            assert blob == O.compress(walk, **kw)
            assert np.array_equal(bits(S.decompress(blob)), bits(O.decompress(blob)))

    def test_big_chunk_bitflips(self):
        rng = np.random.default_rng(99)
        f = np.cumsum(rng.normal(0, 1, 200_000)).astype(np.float32)
        blob = bytearray(S.compress(f, eb=0.02, mode="abs", chunk_size=65536))
        h = S.parse_header(bytes(blob))
        p0 = len(blob) - h.payload_bytes
        for pos in (p0 + 100, p0 + h.payload_bytes // 2, len(blob) - 50):
            b2 = bytearray(blob)
            b2[pos] ^= 0x10
            try:
                want, werr = O.decompress(bytes(b2)), None
            except O.OracleError as e:
                want, werr = None, e
            if werr is None:
                assert np.array_equal(bits(S.decompress(bytes(b2))), bits(want))
            else:
                with pytest.raises(S.SdqzError) as ei:
                    S.decompress(bytes(b2))
                assert str(ei.value) == str(werr)


class TestHostStaging:
    """Host-buffer copies through the pinned staging window (256 MB): a pageable
    field larger than the window uploads in two windows and gives the same
    archive as the device-resident field; the archive round-trips through bytes."""

    def test_pageable_upload_two_windows(self):
        n = 80_000_000                                   # 320 MB fp32 > one staging window
        x = np.linspace(0.0, 40.0, n, dtype=np.float64)
        f = (np.sin(x) + 0.25 * np.sin(7.3 * x)).astype(np.float32)
        blob = S.compress(f, eb=1e-3, mode="abs")        # pageable numpy -> sdqz_upload
        t = torch.from_numpy(f).cuda()
        dev = S.compress_device(t, eb=1e-3, mode="abs")
        assert blob == dev.to_bytes()
        out = S.decompress(blob)
        err = np.abs(out.astype(np.float64) - f.astype(np.float64)).max()
        assert err <= 1e-3 * (1 + 1e-9) + 2 * np.spacing(np.float32(1.25))


class TestGenericShapes:
    """Non-default block shapes run the thread-per-block kernels
    (dq_blocks_kernel / rq_blocks_kernel, row f4): archive bytes and
    decompressed bits equal the oracle's, including partial edge blocks,
    outliers, the int32 magnitude guard (fp64 replay of the block) and
    blocks too large for the per-thread slots (generic kernels)."""

    @pytest.mark.parametrize("dims,block", [
        ((37, 45, 70), (16, 16, 16)), ((37, 45, 70), (4, 4, 4)), ((30, 41, 66), (2, 8, 32)),
        ((19, 23, 130), (1, 1, 64)), ((33, 40, 50), (5, 3, 7)), ((20, 20, 40), (3, 40, 40)),
        ((300, 257), (32, 32)), ((300, 257), (4, 64)), ((129, 130), (1, 7)), ((64, 700), (2, 1000)),
        ((100_003,), (256,)), ((100_003,), (16,)), ((100_003,), (1,)), ((70_001,), (70_000,)),
    ])
    def test_shapes(self, dims, block):
        f = S.generate_field("smooth", dims, seed=len(dims) + block[0]).astype(np.float32)
        f.reshape(-1)[::97] += np.float32(5.0)          # outliers
        for kw in (dict(eb=1e-4, mode="valrel"), dict(eb=0.02, mode="abs", cap=64)):
            blob = S.compress(f, block_shape=block, **kw)
            assert blob == O.compress(f, block_shape=block, **kw)
            assert np.array_equal(bits(S.decompress(blob)), bits(O.decompress(blob)))

    @pytest.mark.parametrize("block", [(16, 16, 16), (2, 8, 40), (8, 40)])
    def test_wide_prequant_range(self, block):
        """valrel on a field far from zero: max|x| / 2eb >= 2^27, so the strip
        dual-quant takes its fp64 path (the int32 one needs every |q| < 2^27)."""
        dims = (40, 41, 90) if len(block) == 3 else (300, 257)
        f = S.generate_field("smooth", dims, seed=9).astype(np.float32) + np.float32(3e4)
        for eb in (1e-7, 1e-5):
            blob = S.compress(f, eb=eb, mode="valrel", block_shape=block)
            assert blob == O.compress(f, eb=eb, mode="valrel", block_shape=block)
            assert np.array_equal(bits(S.decompress(blob)), bits(O.decompress(blob)))

    def test_random_strip_shapes(self):
        """Seeded sweep over the strip / row kernels' geometry: block widths
        below, at and above 32 (one and several lane segments, strips of
        32 // bx blocks with idle lanes), 1-row / 1-plane blocks, fields not a
        multiple of the block, fp32 / fp64, valrel / abs, sprinkled outliers."""
        rng = np.random.default_rng(2024)
        for case in range(24):
            nd = 2 + case % 2
            block = tuple(int(v) for v in rng.choice([1, 2, 3, 5, 8, 16], size=nd - 1)) + \
                (int(rng.choice([3, 7, 12, 31, 32, 33, 40, 64, 100])),)
            dims = tuple(int(b * rng.integers(1, 4) + rng.integers(0, b + 1)) for b in block)
            dims = tuple(max(2, d) for d in dims[:-1]) + (max(3, dims[-1]),)
            dtype = np.float64 if case % 3 == 0 else np.float32
            f = S.generate_field("smooth", dims, seed=case).astype(dtype)
            f.reshape(-1)[rng.integers(0, f.size, size=max(1, f.size // 50))] += dtype(7.0)
            kw = dict(eb=1e-4, mode="valrel") if case % 2 == 0 else dict(eb=0.01, mode="abs", cap=256)
            blob = S.compress(f, block_shape=block, **kw)
            assert blob == O.compress(f, block_shape=block, **kw), (dims, block, dtype, kw)
            assert np.array_equal(bits(S.decompress(blob)), bits(O.decompress(blob))), (dims, block, dtype, kw)

    def test_guard_and_f64(self):
        rng = np.random.default_rng(3)
        f = (rng.normal(0, 1, (24, 24, 24)) * 1e6).astype(np.float64)   # |F| far past 2^28 at eb 1e-3
        for block in ((6, 6, 6), (12, 2, 3)):
            blob = S.compress(f, eb=1e-3, mode="abs", block_shape=block)
            assert blob == O.compress(f, eb=1e-3, mode="abs", block_shape=block)
            assert np.array_equal(bits(S.decompress(blob)), bits(O.decompress(blob)))
        # 1D blocks >= 32: outlier values past 2^29 switch the warp-scan reconstruct to int64
        g = np.cumsum(rng.normal(0, 1, 20_000)) * 1e7
        for block in ((64,), (200,)):
            blob = S.compress(g, eb=1e-3, mode="abs", block_shape=block)
            assert blob == O.compress(g, eb=1e-3, mode="abs", block_shape=block)
            assert np.array_equal(bits(S.decompress(blob)), bits(O.decompress(blob)))


@pytest.mark.gpu
@pytest.mark.parametrize("dims,block", [((33, 70, 90), None), ((300, 700), None), ((250_001,), None),
                                        ((40, 48, 64), (16, 16, 16)), ((120, 200), (4, 64))])
def test_graph_replay_bit_exact(dims, block):
    """Repeated calls with the same geometry replay the captured CUDA graphs
    (the decompress graph carries the forked outlier-index branch): every
    replay's archive and output equal the oracle's."""
    from paper_2007_09625_b200 import _lib
    f = S.generate_field("smooth", dims, seed=11).astype(np.float32)
    f.reshape(-1)[::61] += np.float32(9.0)
    kw = dict(eb=1e-4, mode="valrel", block_shape=block)
    ref = O.compress(f, **kw)
    want = bits(O.decompress(ref))
    ctx = _lib.context()
    r0 = ctx.graph_replays
    for _ in range(4):
        blob = S.compress(f, **kw)
        assert blob == ref
        assert np.array_equal(bits(S.decompress(blob)), want)
    if not os.environ.get("SDQZ_NO_GRAPH"):
        assert ctx.graph_replays > r0

