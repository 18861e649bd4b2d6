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
from paper_2007_09625_b200 import sharded
from paper_2007_09625_b200.sharded import Book


class OracleShardOps:
    """Checker backend: the oracle's stages behind the DeviceShardOps interface."""

    device = torch.device("cpu")

    def field(self, local):
        a = np.ascontiguousarray(local)
        dt = a.dtype if a.dtype in (np.float32, np.float64) else np.dtype(np.float64)
        a = a.astype(dt, copy=False).reshape(-1)
        return torch.from_numpy(a.copy()), np.dtype(dt)

    def describe(self, t, dt):
        vmin, vmax, nf, _ = O.describe(t.numpy())
        return vmin, vmax, nf

    def quantize(self, t, dt, local_dims, cfg):
        codes, oi, ov = O.dualquant(t.numpy(), local_dims, cfg.eb, cfg.cap, cfg.block_shape)
        self._out = (oi, ov)
        c16 = torch.from_numpy(codes.astype(np.uint16).view(np.int16).copy())
        return c16, torch.from_numpy(O.histogram(codes, cfg.cap)), False

    def codebook(self, hist, cap):
        bw = O.tree_bitwidths(hist.numpy())
        book = O.canonical_book(bw)
        return Book(bw.astype(np.uint8), book.unit, int(book.max_bw), book)

    def deflate(self, codes, chunk, book, cap):
        c = codes.numpy().view(np.uint16).astype(np.uint32)
        bits, payload = O.deflate(O.encode(c, book.handle), chunk)
        return (torch.from_numpy(bits.view(np.int32).copy()),
                torch.from_numpy(np.frombuffer(payload, np.uint8).copy()))

    def outliers(self, t, dt, codes, eb):
        oi, ov = self._out
        rec = np.empty((oi.size, 2), np.int64)
        rec[:, 0] = oi.astype(np.int64)
        rec[:, 1] = ov.astype(np.float64).view(np.int64)
        return torch.from_numpy(rec.reshape(-1))

    def inflate(self, payload, chunk_bits, chunk, n_codes, bitwidths):
        book = O.canonical_book(bitwidths)
        return O.inflate(chunk_bits, payload.tobytes(), chunk, book, n_codes)

    def reconstruct(self, codes, idx, vals, local_dims, cfg, dtype):
        n = math.prod(local_dims)
        O.validate_quant(codes, idx, vals, n, cfg.cap)
        v = O.reconstruct(codes, idx, vals, local_dims, cfg.eb, cfg.cap, cfg.block_shape)
        return v.reshape(local_dims).astype(dtype)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, backend, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops = OracleShardOps() if backend == "oracle" else None
        data, dims, rows, kw = case
        r0 = sum(rows[:rank])
        local = data.reshape(dims)[r0: r0 + rows[rank]] if len(dims) > 1 else data[r0: r0 + rows[rank]]
        blob = sharded.compress_sharded(local, dims, ops=ops, **kw)
        slab = sharded.decompress_sharded(blob, rows=rows, ops=ops)
        q.put((rank, blob, slab))
    except Exception as e:  # surfaced by the parent
        q.put((rank, e, None))
    finally:
        dist.destroy_process_group()


def run_sharded(case, world, backend="oracle"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, backend, q)) for r in range(world)]
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
]


@pytest.mark.parametrize("name,dims,rows,kw", CASES, ids=[c[0] for c in CASES])
def test_sharded_archive_equals_single_field(name, dims, rows, kw):
    data = _smooth(dims)
    if name.startswith("3d-cap64"):
        data = data + np.random.default_rng(3).normal(0, 0.3, data.shape).astype(np.float32)
    ref = O.compress(data, dims, **kw)
    blobs, slabs = run_sharded((data.reshape(-1), dims, rows, kw), len(rows))
    for b in blobs:
        assert b == ref
    dec = O.decompress(ref)
    got = np.concatenate([s.reshape((-1,) + tuple(dims[1:])) for s in slabs], axis=0)
    assert np.array_equal(got.reshape(dec.shape).view(np.uint32), dec.view(np.uint32))


def test_slab_rows_split():
    assert sharded.slab_rows(100, 8, 2) == [56, 44]
    assert sharded.slab_rows(2048, 8, 8) == [256] * 8
    assert sum(sharded.slab_rows(13, 8, 4)) == 13


def test_misaligned_slab_rejected():
    dims = (20, 6, 6)
    with pytest.raises(Exception, match="multiple of the block extent"):
        run_sharded((_smooth(dims).reshape(-1), dims, [7, 13], dict(eb=1e-3)), 2)


@pytest.mark.gpu
def test_sharded_device_two_ranks_one_gpu():
    dims = (24, 40, 56)
    kw = dict(eb=1e-4, mode="valrel", chunk_size=1024)
    data = _smooth(dims)
    ref = O.compress(data, dims, **kw)
    blobs, slabs = run_sharded((data.reshape(-1), dims, [8, 16], kw), 2, backend="device")
    assert blobs[0] == ref and blobs[1] == ref
    got = np.concatenate(slabs, axis=0)
    assert np.array_equal(got.view(np.uint32), O.decompress(ref).view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("name,dims,rows,kw", CASES, ids=[c[0] for c in CASES])
def test_sharded_device_cases(name, dims, rows, kw):
    """Every protocol case through the device backend (sdqz_decompress_slab):
    straddling chunks, a chunk spanning three slabs, an empty slab, outliers."""
    data = _smooth(dims)
    if name.startswith("3d-cap64"):
        data = data + np.random.default_rng(3).normal(0, 0.3, data.shape).astype(np.float32)
    ref = O.compress(data, dims, **kw)
    blobs, slabs = run_sharded((data.reshape(-1), dims, rows, kw), len(rows), backend="device")
    for b in blobs:
        assert b == ref
    dec = O.decompress(ref)
    got = np.concatenate([s.reshape((-1,) + tuple(dims[1:])) for s in slabs], axis=0)
    assert np.array_equal(got.reshape(dec.shape).view(np.uint32), dec.view(np.uint32))
