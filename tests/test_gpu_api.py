"""Device-API behaviour: archive handles, argument ranges, per-device contexts."""

from __future__ import annotations

import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2007_09625_b200 as S  # noqa: E402
from oracle import sdqz_oracle as O  # noqa: E402
from paper_2007_09625_b200.pipeline import CompressPlan, DecompressPlan  # noqa: E402


def fields():
    a = S.generate_field("smooth", (24, 40, 56), seed=1).astype(np.float32)
    b = S.generate_field("smooth", (30, 20, 44), seed=2).astype(np.float32)
    return a, b


def test_stale_device_archive_is_refused():
    a, b = fields()
    da = S.compress_device(torch.from_numpy(a).cuda(), eb=1e-4, mode="valrel")
    blob_a = da.to_bytes()
    assert blob_a == O.compress(a, eb=1e-4, mode="valrel")
    db = S.compress_device(torch.from_numpy(b).cuda(), eb=1e-4, mode="valrel")
    assert not da.valid and db.valid
    with pytest.raises(S.SdqzError, match="stale device archive"):
        da.to_bytes()
    with pytest.raises(S.SdqzError, match="stale device archive"):
        S.decompress_device(da)
    assert db.to_bytes() == O.compress(b, eb=1e-4, mode="valrel")
    out = S.decompress_device(db).cpu().numpy()
    assert np.array_equal(out.view(np.uint32), O.decompress(db.to_bytes()).view(np.uint32))


def test_plan_headers_are_per_run():
    a, b = fields()
    pa = CompressPlan(torch.from_numpy(a).cuda(), a.shape, eb=1e-4, mode="valrel")
    pb = CompressPlan(torch.from_numpy(b).cuda(), b.shape, eb=1e-4, mode="valrel")
    da = pa.run()
    ha = (da.header.n_outliers, da.header.payload_bytes)
    db = pb.run()
    assert (da.header.n_outliers, da.header.payload_bytes) == ha
    assert db.header.dims[0] == 30 and da.header.dims[0] == 24
    dp = DecompressPlan(db)
    out = dp.run().cpu().numpy()
    assert np.array_equal(out.view(np.uint32), O.decompress(db.to_bytes()).reshape(-1).view(np.uint32))
    with pytest.raises(S.SdqzError, match="stale"):
        DecompressPlan(da).run()


def test_chunk_size_beyond_u32_is_not_truncated():
    a = np.linspace(-1, 1, 1000, dtype=np.float32)
    with pytest.raises(struct.error):
        S.compress(a, eb=1e-3, chunk_size=2**32)
    with pytest.raises(struct.error):
        S.compress(a, eb=1e-3, chunk_size=2**32 + 256)
    # errors the reference raises earlier still win
    with pytest.raises(S.SdqzError, match="NaN"):
        S.compress(np.array([1.0, np.nan], np.float32), eb=1e-3, chunk_size=2**32)


def test_second_device_context_if_present():
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU")
    a, _ = fields()
    blobs = []
    for d in range(2):
        with torch.cuda.device(d):
            blobs.append(S.compress(a, eb=1e-4, mode="valrel"))
    assert blobs[0] == blobs[1]


@pytest.mark.gpu
@pytest.mark.parametrize("shape,mode,eb", [((40, 56, 24), "valrel", 1e-4), ((1800, 36), "abs", 0.05),
                                           ((100003,), "valrel", 1e-3)])
def test_host_buffer_path_matches(shape, mode, eb):
    """sdqz_compress_host / sdqz_decompress_host / sdqz_quality_host (the CLI's
    torch-free path) produce the same archive, field and scores."""
    import paper_2007_09625_b200 as S
    from paper_2007_09625_b200 import metrics, pipeline
    f = S.generate_field("smooth", shape, seed=3).astype(np.float32)
    blob = S.compress(f, eb=eb, mode=mode)
    assert pipeline.compress_host(f, eb=eb, mode=mode) == blob
    out = pipeline.decompress_host(blob)
    assert out.shape == shape and np.array_equal(out.view(np.uint32), S.decompress(blob).view(np.uint32))
    assert metrics.quality_host(f, out) == metrics.quality(f, out)


@pytest.mark.gpu
def test_host_buffer_path_errors():
    import paper_2007_09625_b200 as S
    from paper_2007_09625_b200 import pipeline
    bad = np.ones(64, np.float32)
    bad[3] = np.nan
    with pytest.raises(S.SdqzError, match="NaN"):
        pipeline.compress_host(bad, eb=0.1)
    with pytest.raises(S.ArchiveFormatError, match="bad magic"):
        pipeline.decompress_host(b"XXXX" + bytes(100))
    blob = bytearray(S.compress(S.generate_field("smooth", (32, 32), seed=1).astype(np.float32), eb=1e-3))
    with pytest.raises(S.ArchiveFormatError):
        pipeline.decompress_host(bytes(blob[:60]))


@pytest.mark.gpu
@pytest.mark.parametrize("shape,kw,want_fused", [
    ((40, 56, 24), dict(eb=1e-4, mode="valrel"), True),                 # 3D block kernel
    ((300, 256), dict(eb=1e-3, mode="valrel"), True),                   # vectorised 2D
    ((100003,), dict(eb=1e-4, mode="valrel"), True),                    # 1D records kernel
    ((30, 33, 20), dict(eb=0.02, block_shape=(4, 3, 2)), False),        # generic shape: separate pass
])
def test_fused_quality_matches_separate(shape, kw, want_fused):
    """sdqz_decompress_quality: the same field as decompress_device and the
    same scores as quality() (sum of squares up to summation order)."""
    from paper_2007_09625_b200 import metrics, pipeline
    f = S.generate_field("smooth", shape, seed=5).astype(np.float32)
    t = torch.from_numpy(f).cuda()
    dev = S.compress_device(t, **kw)
    ref = S.decompress_device(dev).clone()
    out, q5, fused = pipeline.decompress_quality(dev, t)
    assert fused == want_fused
    assert torch.equal(out.view(torch.int32), ref.view(torch.int32))
    q = metrics.quality(t, ref)
    qf = metrics._report(q5, f.size)
    assert qf.max_abs_error == q.max_abs_error and qf.value_range == q.value_range
    assert qf.rmse == pytest.approx(q.rmse, rel=1e-12)
    rows = S.rd_sweep(f, S.describe_field(f, shape), [S.ErrorBoundSpec(kw.get("mode", "abs"), kw["eb"])],
                      **({"chunk_size": None} if "block_shape" not in kw else {}))
    assert rows[0].error is None or "block" in rows[0].error


@pytest.mark.gpu
def test_compress_described_matches():
    """sdqz_compress_described (rd_sweep's K1 reuse) gives the same archives,
    and the same errors, as sdqz_compress."""
    from paper_2007_09625_b200 import _device
    f = S.generate_field("smooth", (33, 40, 48), seed=6).astype(np.float32)
    t = torch.from_numpy(f).cuda().reshape(-1)
    stats = _device.describe(t, np.dtype(np.float32))
    for eb in (1e-2, 1e-3, 1e-4, 1e-5):
        want = S.compress(f, eb=eb, mode="valrel")
        assert S.compress_device(t, f.shape, eb=eb, mode="valrel", stats=stats).to_bytes() == want
    bad = f.copy()
    bad[3, 4, 5] = np.inf
    tb = torch.from_numpy(bad).cuda().reshape(-1)
    with pytest.raises(S.SdqzError, match="NaN/Inf"):
        S.compress_device(tb, bad.shape, eb=1e-3, mode="valrel", stats=_device.describe(tb, np.dtype(np.float32)))
    rows = S.rd_sweep(f, S.describe_field(f, f.shape), [S.ErrorBoundSpec("valrel", e) for e in (1e-2, 1e-4)])
    assert [r.n_outliers for r in rows] == [S.parse_header(S.compress(f, eb=e, mode="valrel")).n_outliers
                                           for e in (1e-2, 1e-4)]
