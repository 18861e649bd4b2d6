"""Multi-process slab sharding (paper_2007_09625_b200/sharded.py).

CPU: world_size 2/3 gloo groups drive the exchange protocol with a checker
backend built on the oracle (the per-slab compute is the oracle's, so these
tests pin the protocol: chunk ownership, straddling chunks, global histogram,
assembly); the sharded archive must equal the oracle's single-field archive
byte for byte, and the sharded decompress must equal the oracle's.
GPU: the same protocol with the device backend (libsdqz_cuda.so) in 2
processes sharing cuda:0 over gloo.
"""

from __future__ import annotations

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sdqz_oracle as O
import paper_2007_09625_b200 as S
from paper_2007_09625_b200 import sharded


class OracleShardOps:
    """Checker backend: the oracle's stages behind the DeviceShardOps interface
    (describe -> quantize -> head -> encode; decompress_slab)."""

    device = torch.device("cpu")

    def field(self, local):
        a = np.ascontiguousarray(local)
        dt = a.dtype if a.dtype in (np.float32, np.float64) else np.dtype(np.float64)
        a = a.astype(dt, copy=False).reshape(-1)
        return torch.from_numpy(a.copy()), np.dtype(dt)

    def describe(self, t, dt):
        if t.numel() == 0:
            return torch.tensor([-np.inf, -np.inf, 0.0], dtype=torch.float64)
        vmin, vmax, nf, _ = O.describe(t.numpy())
        return torch.tensor([-vmin, vmax, 1.0 if nf else 0.0], dtype=torch.float64)

    def quantize(self, t, dt, local_dims, block, mode, eb, cap, rng):
        r = rng.numpy()
        self.eb = O.resolve_eb(mode, eb, -r[0], r[1], r[2] > 0)
        self.cap = cap
        if t.numel():
            codes, oi, ov = O.dualquant(t.numpy(), local_dims, self.eb, cap, block)
        else:
            codes, oi, ov = np.zeros(0, np.uint32), np.zeros(0, np.uint64), np.zeros(0)
        self.codes, self.oi, self.ov = codes.reshape(-1), oi, ov
        return torch.from_numpy(O.histogram(self.codes, cap))

    def head(self, count):
        return torch.from_numpy(self.codes[:count].astype(np.uint16).view(np.int16).copy())

    def encode(self, hist, chunk, head, tail, idx_base):
        book = O.canonical_book(O.tree_bitwidths(hist.numpy()))
        parts = [self.codes[head:]]
        if tail is not None:
            parts.append(tail.numpy().view(np.uint16).astype(np.uint32))
        packed = np.concatenate(parts)
        if packed.size:
            bits, payload = O.deflate(O.encode(packed, book), chunk)
        else:
            bits, payload = np.zeros(0, np.uint32), b""
        rec = np.empty((self.oi.size, 2), np.int64)
        rec[:, 0] = self.oi.astype(np.int64) + idx_base
        rec[:, 1] = self.ov.astype(np.float64).view(np.int64)
        pay = np.zeros(len(payload) + 64, np.uint8)
        pay[: len(payload)] = np.frombuffer(payload, np.uint8)
        bw = O.tree_bitwidths(hist.numpy()).astype(np.uint8)
        sec = {"bitwidths": torch.from_numpy(bw), "outliers": torch.from_numpy(rec.reshape(-1)),
               "chunk_bits": torch.from_numpy(bits.astype(np.uint32).view(np.int32).copy()),
               "payload": torch.from_numpy(pay), "payload_bytes": len(payload)}
        sizes = {"n_chunks": int(bits.size), "payload_bytes": len(payload), "n_outliers": int(self.oi.size),
                 "unit_width": int(book.unit), "eb_resolved": float(self.eb)}
        return sizes, sec

    def decompress_slab(self, h, bw, rec, k, idx_base, bits, payload, payload_bytes, n_range, lo, local_dims):
        book = O.canonical_book(bw.numpy())
        codes = O.inflate(bits.numpy().view(np.uint32), payload.numpy()[:payload_bytes].tobytes(),
                          h.chunk_size, book, n_range)
        n = math.prod(local_dims)
        codes = np.asarray(codes)[lo: lo + n]
        r = rec.numpy().reshape(-1, 2)[:k]
        idx = r[:, 0].astype(np.uint64) - np.uint64(idx_base)
        vals = r[:, 1].view(np.float64)
        O.validate_quant(codes, idx, vals, n, h.cap)
        v = O.reconstruct(codes, idx, vals, local_dims, h.eb_resolved, h.cap, h.block_shape[: h.ndims])
        return torch.from_numpy(v.reshape(local_dims).astype(h.np_dtype))

    def upload(self, a):
        return torch.from_numpy(np.ascontiguousarray(a).copy())

    def to_numpy(self, t):
        return t.numpy()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, backend, q, tmpdir, pg="gloo"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if pg == "nccl":   # the box's backend: collectives on CUDA tensors (one rank per GPU)
        import torch
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops = OracleShardOps() if backend == "oracle" else None
        data, dims, rows, kw = case
        r0 = sum(rows[:rank])
        local = data.reshape(dims)[r0: r0 + rows[rank]] if len(dims) > 1 else data[r0: r0 + rows[rank]]
        ar = sharded.compress_sharded_device(local, dims, ops=ops, **kw)
        blob = ar.to_bytes()
        path = os.path.join(tmpdir, "sharded.sdqz")
        ar.write(path)
        with open(path, "rb") as f:
            written = f.read()
        gathered = ar.gather(root=0)
        slab = sharded.decompress_sharded(blob, rows=rows, ops=ops)             # bytes path
        slab2 = sharded.decompress_sharded(ar, ops=ops)                          # in place (or fallback)
        q.put((rank, (blob, written, gathered), (slab, slab2)))
    except Exception as e:  # surfaced by the parent
        q.put((rank, e, None))
    finally:
        dist.destroy_process_group()


def run_sharded(case, world, backend="oracle", pg="gloo"):
    import tempfile
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    tmpdir = tempfile.mkdtemp(prefix="sdqz_sharded_")
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, backend, q, tmpdir, pg))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(world):
        r, blob, slab = q.get(timeout=300)
        res[r] = (blob, slab)
    for p in procs:
        p.join(60)
    for r in range(world):
        if isinstance(res[r][0], Exception):
            raise res[r][0]
    return [res[r][0] for r in range(world)], [res[r][1] for r in range(world)]


def _smooth(dims, seed=1):
    return O.smooth_field(dims, seed).astype(np.float32)


CASES = [
    # dims, rows per rank, kwargs: straddling chunks (rows*inner not chunk-aligned)
    ("3d-straddle", (20, 30, 36), [8, 12], dict(eb=1e-3, mode="valrel", chunk_size=256)),
    ("3d-3ranks", (40, 17, 9), [16, 8, 16], dict(eb=1e-4, mode="valrel", chunk_size=1000)),
    # a chunk spanning three slabs (slabs smaller than one chunk)
    ("1d-span3", (3000,), [320, 640, 2040], dict(eb=1e-3, mode="abs", chunk_size=2048)),
    ("2d-default-chunk", (70, 50), [32, 38], dict(eb=1e-4, mode="valrel")),
    ("2d-empty-slab", (40, 33), [32, 0, 8], dict(eb=1e-2, mode="valrel", chunk_size=300)),
    ("3d-cap64-outliers", (16, 12, 20), [8, 8], dict(eb=1e-5, mode="valrel", cap=64, chunk_size=512)),
    # slabs on chunk boundaries (the 2048x2048x1024 layout in miniature): in-place decompress
    ("3d-chunk-aligned", (32, 16, 32), [8, 16, 8], dict(eb=1e-4, mode="valrel", chunk_size=512)),
    ("3d-aligned-4ranks", (64, 24, 40), [16, 16, 16, 16], dict(eb=1e-4, mode="valrel", chunk_size=3840)),
]


def _field(name, dims):
    data = _smooth(dims)
    if name.startswith("3d-cap64"):
        data = data + np.random.default_rng(3).normal(0, 0.3, data.shape).astype(np.float32)
    return data


def _check(ref, dims, outs, slabs):
    """Every assembly path gives the single-field archive; both decompress
    paths give its decompressed field."""
    dec = O.decompress(ref)
    for r, (blob, written, gathered) in enumerate(outs):
        assert blob == ref
        assert written == ref
        assert gathered == (ref if r == 0 else None)
    for k in range(2):
        got = np.concatenate([np.asarray(s[k]).reshape((-1,) + tuple(dims[1:])) for s in slabs], axis=0)
        assert np.array_equal(got.reshape(dec.shape).view(np.uint32), dec.view(np.uint32)), k


@pytest.mark.parametrize("name,dims,rows,kw", CASES, ids=[c[0] for c in CASES])
def test_sharded_archive_equals_single_field(name, dims, rows, kw):
    data = _field(name, dims)
    ref = O.compress(data, dims, **kw)
    outs, slabs = run_sharded((data.reshape(-1), dims, rows, kw), len(rows))
    _check(ref, dims, outs, slabs)


def test_slab_rows_split():
    assert sharded.slab_rows(100, 8, 2) == [56, 44]
    assert sharded.slab_rows(2048, 8, 8) == [256] * 8
    assert sum(sharded.slab_rows(13, 8, 4)) == 13


def test_misaligned_slab_rejected():
    dims = (20, 6, 6)
    with pytest.raises(Exception, match="multiple of the block extent"):
        run_sharded((_smooth(dims).reshape(-1), dims, [7, 13], dict(eb=1e-3)), 2)


def _decompress_worker(rank, world, port, blob, rows, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sharded.decompress_sharded(blob, rows=rows, ops=OracleShardOps())
        q.put((rank, None))
    except Exception as e:
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def test_decompress_misaligned_rows_rejected():
    """Caller-supplied slab heights must be whole block rows (as compress
    requires), or the slab's block grid would not match the encoder's."""
    dims = (20, 6, 6)
    blob = O.compress(_smooth(dims), dims, eb=1e-3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_decompress_worker, args=(r, 2, port, blob, [7, 13], q)) for r in range(2)]
    for p in procs:
        p.start()
    errs = [q.get(timeout=120)[1] for _ in range(2)]
    for p in procs:
        p.join(60)
    assert all(isinstance(e, Exception) and "multiple of the block extent" in str(e) for e in errs)


def test_record_checks():
    with pytest.raises(S.ArchiveFormatError, match="not strictly ascending"):
        sharded._validate_records(np.array([3, 3], np.uint64), 10)
    with pytest.raises(S.ArchiveFormatError, match="out of range"):
        sharded._validate_records(np.array([3, 10], np.uint64), 10)


@pytest.mark.gpu
@pytest.mark.parametrize("name,dims,rows,kw", CASES, ids=[c[0] for c in CASES])
def test_sharded_device_cases(name, dims, rows, kw):
    """Every protocol case through the fused device pipeline (sdqz_shard_*,
    sdqz_decompress_slab), ranks sharing cuda:0 over gloo: straddling chunks,
    a chunk spanning three slabs, an empty slab, outliers, in-place decompress."""
    data = _field(name, dims)
    ref = O.compress(data, dims, **kw)
    outs, slabs = run_sharded((data.reshape(-1), dims, rows, kw), len(rows), backend="device")
    _check(ref, dims, outs, slabs)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["3d-straddle", "2d-default-chunk", "1d-span3"])
def test_sharded_nccl_backend(name):
    """The NCCL code path (collectives on CUDA tensors, as on the multi-GPU box)
    with one rank per GPU available here: the whole field as one slab."""
    import torch
    if not torch.cuda.is_available() or not torch.distributed.is_nccl_available():
        pytest.skip("needs CUDA + NCCL")
    world = min(torch.cuda.device_count(), 2)
    _, dims, rows, kw = next(c for c in CASES if c[0] == name)
    data = _field(name, dims)
    ref = O.compress(data, dims, **kw)
    rows = sharded.slab_rows(dims[0], {1: 32, 2: 16, 3: 8}[len(dims)], world)
    outs, slabs = run_sharded((data.reshape(-1), dims, rows, kw), world, backend="device", pg="nccl")
    _check(ref, dims, outs, slabs)
