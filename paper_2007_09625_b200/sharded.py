"""Multi-GPU slab sharding of compress / decompress.

One process per GPU under `torch.distributed` (NCCL over NVLink on the box;
gloo in the CPU tests).  A field is split along axis 0 into slabs of whole
block rows -- Lorenzo blocks are zero-padded and independent
(dualquant.py:81-86, :185-186), and the reference itself decomposes fields
this way for workers > 1 (`_row_slabs`, dualquant.py:230-273) -- so every
slab quantizes exactly as the same rows of the whole field do.  Per rank
there is ONE fused device pipeline (include/sdqz_cuda.h, sdqz_shard_*) in
three phases around three small collectives:

  1. describe the slab -> all-reduce MAX of {-min, max, nonfinite}: the same
     resolved bound on every rank (core.py:161-175), computed on the device;
  2. dual-quant + histogram -> all-reduce SUM of the histogram: every rank
     builds the identical codebook (K3 is deterministic);
  3. encode: chunks of default_chunk_size(N_global) (huffman.py:206-212); a
     rank packs the chunks that START in its slab.  When slab boundaries are
     not chunk boundaries, a straddling chunk's tail codes come from the
     following ranks' heads (< chunk_size codes each, one all-gather).  The
     rank's outlier records carry global indices (slab offset + local).

Assembly is an all-gather of (n_chunks, payload_bytes, n_outliers) only: an
exclusive scan gives every rank the byte offset of each of its sections in
the archive, so the archive exists as a `ShardedArchive` -- every rank's
sections on its own GPU plus the global header -- that is written in
parallel (`write`: each rank writes its own byte ranges of one file),
gathered to one rank (`gather`), or decompressed in place (each rank decodes
the chunks that cover its slab with its outlier records: no collective at
all when slabs start on chunk boundaries, as for the 2048x2048x1024 config).
Concatenating the sections in rank order IS the single-GPU archive (outlier
indices stay ascending), byte for byte.

The per-rank compute goes through `DeviceShardOps`; the exchange protocol
only sees tensors, so the CPU tests drive it with a gloo group and a checker
backend built on the oracle.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from .archive import HEADER_SIZE, ArchiveFormatError, ArchiveHeader, pack_header, parse_header
from .core import ErrorBoundSpec, QuantConfig, SdqzError, _as_dims
from .huffman import default_chunk_size

_RECORD = np.dtype([("index", "<u8"), ("value", "<f8")])


# --------------------------------------------------------------------------
# per-rank compute on this rank's GPU
# --------------------------------------------------------------------------
class DeviceShardOps:
    """The rank's pipeline through the C-ABI (include/sdqz_cuda.h, sdqz_shard_*)."""

    def __init__(self):
        _lib.require_cuda()

    @property
    def device(self):
        torch = _device._torch()
        return torch.device("cuda", torch.cuda.current_device())

    def field(self, local):
        return _device.to_device(_device.as_field(local))

    def describe(self, t, dt):
        """-> float64[3] {-min, max, nonfinite} of the slab (device)."""
        torch = _device._torch()
        r = _device.empty(3, torch.float64)
        _lib.context().call("sdqz_shard_describe", _lib.ptr(t), 0 if dt == np.float32 else 1,
                            int(t.numel()), _lib.ptr(r))
        return r

    def quantize(self, t, dt, local_dims, block, mode, eb, cap, rng):
        """Dual-quant of the slab with the bound resolved from the reduced range
        -> int64[cap] local histogram (device)."""
        torch = _device._torch()
        hist = _device.empty(cap, torch.int64)
        _lib.context().call("sdqz_shard_quantize", _lib.ptr(t), 0 if dt == np.float32 else 1,
                            len(local_dims), _lib.dims3(local_dims), _lib.block3(block),
                            0 if mode == "abs" else 1, float(eb), int(cap), _lib.ptr(rng),
                            _lib.ptr(hist))
        return hist

    def head(self, count: int):
        """The slab's first `count` codes (packed by the previous rank)."""
        torch = _device._torch()
        h = _device.empty(count, torch.int16)
        _lib.context().call("sdqz_shard_head", int(count), _lib.ptr(h))
        return h[:count]

    def encode(self, hist, chunk: int, head: int, tail, idx_base: int):
        """-> (sizes dict, sections dict of device tensors)."""
        torch = _device._torch()
        ctx = _lib.context()
        sz = _lib.ShardSizes()
        tail = tail.contiguous() if tail is not None and tail.numel() else None
        ctx.call("sdqz_shard_encode", _lib.ptr(hist), int(chunk), int(head), _lib.ptr(tail),
                 int(tail.numel()) if tail is not None else 0, int(idx_base), ctypes.byref(sz))
        cap = int(hist.numel())
        sec = {"bitwidths": _device.empty(cap, torch.uint8)[:cap],
               "outliers": _device.empty(2 * sz.n_outliers, torch.int64)[:2 * sz.n_outliers],
               "chunk_bits": _device.zeros(sz.n_chunks + 4, torch.int32)[:sz.n_chunks],
               "payload": _device.empty(sz.payload_bytes + 64, torch.uint8)}
        sec["payload"][sz.payload_bytes:].zero_()
        ctx.call("sdqz_archive_copy", ctx.archive_generation, _lib.ptr(sec["bitwidths"]),
                 _lib.ptr(sec["outliers"]) if sz.n_outliers else None,
                 _lib.ptr(sec["chunk_bits"]) if sz.n_chunks else None, _lib.ptr(sec["payload"]))
        sec["payload_bytes"] = int(sz.payload_bytes)
        sizes = {"n_chunks": int(sz.n_chunks), "payload_bytes": int(sz.payload_bytes),
                 "n_outliers": int(sz.n_outliers), "unit_width": int(sz.unit_width),
                 "eb_resolved": float(sz.eb_resolved)}
        return sizes, sec

    def decompress_slab(self, h: ArchiveHeader, bw, rec, k: int, idx_base: int, bits, payload,
                        payload_bytes: int, n_range: int, lo: int, local_dims):
        """Device-resident slab decompress (sdqz_decompress_slab) from device
        sections -> the slab as a device tensor."""
        torch = _device._torch()
        ch = _header_struct(h)
        ch.n_outliers, ch.n_chunks, ch.payload_bytes = k, int(bits.numel()), payload_bytes
        n = math.prod(local_dims)
        out = _device.empty(n, torch.float32 if h.dtype_code == 0 else torch.float64)
        _lib.context().call("sdqz_decompress_slab", ctypes.byref(ch), _lib.ptr(bw), _lib.ptr(rec), int(k),
                            int(idx_base), _lib.ptr(bits), int(bits.numel()), _lib.ptr(payload),
                            int(payload_bytes), int(n_range), int(lo), _lib.dims3(local_dims), _lib.ptr(out))
        return out[:n].view(*local_dims) if n else out[:0]

    def upload(self, a: np.ndarray):
        return _device.upload(a)

    def to_numpy(self, t):
        return _device.download(t) if t.is_cuda else t.numpy()


def _header_struct(h: ArchiveHeader):
    ch = _lib.Header()
    ch.dtype_code, ch.ndims, ch.eb_mode, ch.unit_width = h.dtype_code, h.ndims, h.eb_mode, h.unit_width
    for a in range(3):
        ch.dims[a] = h.dims[a]
        ch.block[a] = h.block_shape[a]
    ch.eb_resolved, ch.eb_specified, ch.cap, ch.chunk_size = (h.eb_resolved, h.eb_specified, h.cap,
                                                              h.chunk_size)
    return ch


# --------------------------------------------------------------------------
# collectives (tensors live on the group's device: CUDA for NCCL, CPU for gloo)
# --------------------------------------------------------------------------
def _comm_device(group):
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _all_reduce(t, op, group):
    """All-reduce `t` in place (through a comm-device copy when needed)."""
    import torch.distributed as dist
    dev = _comm_device(group)
    if t.device == dev:
        dist.all_reduce(t, op=op, group=group)
        return t
    c = t.to(dev)
    dist.all_reduce(c, op=op, group=group)
    t.copy_(c)
    return t


def _allgather_i64(values, group):
    import torch
    import torch.distributed as dist
    dev = _comm_device(group)
    world = dist.get_world_size(group)
    t = torch.tensor(list(values), dtype=torch.int64, device=dev)
    out = torch.empty(world * t.numel(), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(out, t, group=group)
    return out.view(world, -1).cpu().numpy()


def _allgather_var(t, group):
    """Variable-length 1-D uint8 tensors -> list of per-rank uint8 tensors (comm device)."""
    import torch
    import torch.distributed as dist
    dev = _comm_device(group)
    world = dist.get_world_size(group)
    t = t.reshape(-1).to(dev)
    sizes = _allgather_i64([t.numel()], group)[:, 0]
    m = max(1, int(sizes.max()))
    buf = torch.zeros(m, dtype=torch.uint8, device=dev)
    buf[: t.numel()] = t
    out = torch.empty(world * m, dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(out, buf, group=group)
    out = out.view(world, m)
    return [out[r, : int(sizes[r])] for r in range(world)]


def _as_bytes(t):
    """Any contiguous tensor -> flat uint8 view."""
    import torch
    t = t.contiguous().reshape(-1)
    return t.view(torch.uint8) if t.numel() else t.new_empty(0, dtype=torch.uint8)


def slab_rows(n_rows: int, block0: int, world: int) -> list[int]:
    """Even split of axis 0 into `world` slabs of whole block-rows (rank order)."""
    granules = -(-n_rows // block0)
    base, extra = divmod(granules, world)
    rows, left = [], n_rows
    for r in range(world):
        take = min(left, (base + (1 if r < extra else 0)) * block0)
        rows.append(take)
        left -= take
    return rows


def _check_rows(rows, b0):
    for i, r in enumerate(rows[:-1]):
        if r % b0:
            raise SdqzError(f"slab {i} has {r} rows; every slab but the last must be a "
                            f"multiple of the block extent {b0}")


# --------------------------------------------------------------------------
# the sharded archive
# --------------------------------------------------------------------------
@dataclass
class ShardedArchive:
    """One archive whose sections are spread over the ranks of `group`.

    `header` is the global header (identical on every rank); `rank_sizes[r]`
    = (n_chunks, payload_bytes, n_outliers) of rank r, so every rank knows
    where each rank's sections sit in the serialized archive; `sections` are
    this rank's (device) tensors."""

    header: ArchiveHeader
    bitwidths: np.ndarray
    rows: list
    rank_sizes: np.ndarray
    sections: dict
    group: object
    ops: object

    @property
    def nbytes(self) -> int:
        return self.header.total_bytes

    def layout(self, r: int):
        """Byte offsets in the archive of rank r's outliers, chunk bits, payload."""
        h = self.header
        rs = self.rank_sizes
        o_rec = HEADER_SIZE + h.cap + 16 * int(rs[:r, 2].sum())
        o_bits = HEADER_SIZE + h.cap + 16 * h.n_outliers + 4 * int(rs[:r, 0].sum())
        o_pay = (HEADER_SIZE + h.cap + 16 * h.n_outliers + 4 * h.n_chunks + int(rs[:r, 1].sum()))
        return o_rec, o_bits, o_pay

    def _local_parts(self):
        s = self.sections
        return (_as_bytes(s["outliers"]), _as_bytes(s["chunk_bits"]),
                s["payload"][: s["payload_bytes"]])

    def head_bytes(self) -> bytes:
        return pack_header(self.header) + np.ascontiguousarray(self.bitwidths, np.uint8).tobytes()

    def to_bytes(self) -> bytes:
        """The whole archive on every rank (all-gather of the sections)."""
        parts = [_allgather_var(p, self.group) for p in self._local_parts()]
        body = [x.cpu().numpy().tobytes() for sec in parts for x in sec]
        return self.head_bytes() + b"".join(body)

    def gather(self, root: int = 0):
        """The whole archive on `root` (None elsewhere)."""
        import torch.distributed as dist
        rank = dist.get_rank(self.group)
        parts = [_allgather_var(p, self.group) for p in self._local_parts()]
        if rank != root:
            return None
        return self.head_bytes() + b"".join(x.cpu().numpy().tobytes() for sec in parts for x in sec)

    def write(self, path: str) -> int:
        """Every rank writes its own sections at their offsets of one file
        (rank 0 also the header and bitwidths): parallel assembly, no data
        exchange.  Returns the archive size."""
        import torch.distributed as dist
        rank = dist.get_rank(self.group)
        if rank == 0:
            with open(path, "wb") as f:
                f.truncate(self.nbytes)
                f.write(self.head_bytes())
        dist.barrier(group=self.group)
        fd = os.open(path, os.O_WRONLY)
        try:
            for off, part in zip(self.layout(rank), self._local_parts()):
                if part.numel():
                    os.pwrite(fd, self.ops.to_numpy(part).tobytes(), off)
        finally:
            os.close(fd)
        dist.barrier(group=self.group)
        return self.nbytes


# --------------------------------------------------------------------------
# compress
# --------------------------------------------------------------------------
def compress_sharded_device(local, dims, *, eb: float, mode: str = "abs", cap: int = 1024,
                            block_shape=None, chunk_size: int | None = None, group=None,
                            ops=None) -> ShardedArchive:
    """Compress a field whose axis-0 slabs are spread over the ranks of `group`
    (`local` = this rank's rows, in rank order; `dims` = the GLOBAL dims)."""
    import torch
    import torch.distributed as dist

    ops = ops or DeviceShardOps()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dims = _as_dims(dims)
    if len(dims) > 3:
        raise SdqzError(f"rank {len(dims)} fields are not supported (1-3)")
    nd, inner, n_global = len(dims), math.prod(dims[1:]), math.prod(dims)
    t, dt = ops.field(local)
    n_local = int(t.numel())
    if n_local % inner:
        raise SdqzError(f"slab of {n_local} values is not a whole number of rows of {dims}")
    rows_local = n_local // inner
    meta = _allgather_i64([rows_local, 0 if dt == np.float32 else 1], group)
    rows = [int(x) for x in meta[:, 0]]
    if len(set(int(x) for x in meta[:, 1])) != 1:
        raise SdqzError("all slabs must share one dtype")
    if sum(rows) != dims[0]:
        raise SdqzError(f"slabs cover {sum(rows)} rows but dims {'x'.join(map(str, dims))} "
                        f"require {dims[0]}")
    ErrorBoundSpec(mode, eb)
    cfg = QuantConfig.for_rank(1.0, nd, cap=cap, block_shape=block_shape)   # validates cap/block
    _check_rows(rows, cfg.block_shape[0])
    if chunk_size is not None and chunk_size < 1:
        raise SdqzError("chunk_size must be >= 1")
    cs = int(chunk_size or default_chunk_size(n_global))
    offs = [sum(rows[:r]) * inner for r in range(world + 1)]
    o = offs[rank]
    local_dims = (rows_local,) + tuple(dims[1:])

    # 1. global range -> the resolved bound (on the device, identical everywhere)
    rng = ops.describe(t, dt)
    _all_reduce(rng, dist.ReduceOp.MAX, group)
    # 2. slab dual-quant; global histogram -> identical codebook
    hist = ops.quantize(t, dt, local_dims, cfg.block_shape, mode, eb, cap, rng)
    _all_reduce(hist, dist.ReduceOp.SUM, group)
    # 3. chunk ownership: a rank packs the chunks that start in its slab; the
    #    codes before its first own chunk start (its head) go to the owner
    heads = [min(-(-offs[r] // cs) * cs, offs[r + 1]) - offs[r] for r in range(world)]
    head = heads[rank]
    tail = None
    if any(heads[1:]):
        hcodes = _allgather_var(_as_bytes(ops.head(head)), group)
        if head < n_local:   # this rank owns chunks: complete the last one
            end = min(-(-offs[rank + 1] // cs) * cs, n_global)
            need = end - offs[rank + 1]
            parts = []
            for r in range(rank + 1, world):
                if need <= 0:
                    break
                hr = hcodes[r].view(torch.int16)
                take = min(need, hr.numel())
                parts.append(hr[:take])
                need -= take
            if need:
                raise SdqzError("internal: straddling chunk not covered by the following slabs")
            if parts:
                tail = torch.cat(parts).to(ops.device)
    sizes, sec = ops.encode(hist, cs, head, tail, o)
    # assembly: sizes only
    g = _allgather_i64([sizes["n_chunks"], sizes["payload_bytes"], sizes["n_outliers"],
                        sizes["unit_width"],
                        int(np.float64(sizes["eb_resolved"]).view(np.int64))], group)
    if len(set(g[:, 3].tolist())) != 1 or len(set(g[:, 4].tolist())) != 1:
        raise SdqzError("internal: ranks disagree on the codebook or the bound")
    n_chunks, p_bytes, n_out = int(g[:, 0].sum()), int(g[:, 1].sum()), int(g[:, 2].sum())
    if n_chunks != -(-n_global // cs):
        raise SdqzError("internal: chunk count mismatch after assembly")
    hdr = ArchiveHeader(
        dtype_code=0 if dt == np.float32 else 1, ndims=nd, eb_mode=0 if mode == "abs" else 1,
        dims=tuple(dims) + (1,) * (3 - nd), eb_resolved=sizes["eb_resolved"], eb_specified=float(eb),
        cap=cap, block_shape=tuple(cfg.block_shape) + (1,) * (3 - nd), chunk_size=cs,
        unit_width=int(g[0, 3]), n_outliers=n_out, n_chunks=n_chunks, payload_bytes=p_bytes)
    bw = ops.to_numpy(sec["bitwidths"]).astype(np.uint8)
    return ShardedArchive(hdr, bw, rows, g[:, :3].copy(), sec, group, ops)


def compress_sharded(local, dims, *, eb: float, mode: str = "abs", cap: int = 1024,
                     block_shape=None, chunk_size: int | None = None, group=None,
                     ops=None) -> bytes:
    """compress_sharded_device + the archive bytes on every rank, identical to
    `compress(whole_field, dims, ...)` on one GPU (pipeline.py:15-39)."""
    return compress_sharded_device(local, dims, eb=eb, mode=mode, cap=cap, block_shape=block_shape,
                                   chunk_size=chunk_size, group=group, ops=ops).to_bytes()


# --------------------------------------------------------------------------
# decompress
# --------------------------------------------------------------------------
def _validate_records(idx: np.ndarray, n: int):
    """archive.deserialize's record checks (archive.py:220-225)."""
    if idx.size:
        if int(idx.max()) >= n:
            raise ArchiveFormatError("outlier index out of range")
        if np.any(np.diff(idx.astype(np.int64)) <= 0):
            raise ArchiveFormatError("outlier indices not strictly ascending")


def decompress_sharded(src, *, group=None, rows: list[int] | None = None, ops=None, device=False):
    """Reconstruct this rank's slab of an archive (pipeline.py:42-58 on a row
    range).  `src` is archive bytes (every rank holds them) or a
    ShardedArchive (each rank holds its own sections).  `rows` gives every
    rank's slab height (default: the archive's own split for a
    ShardedArchive, else an even split in whole block rows); every slab but
    the last must be a whole number of block rows.  Returns the slab shaped
    (rows_r, *dims[1:]) -- a numpy array, or the device tensor if `device`."""
    import torch.distributed as dist

    ops = ops or DeviceShardOps()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if isinstance(src, ShardedArchive):
        if rows is None or list(rows) == list(src.rows):
            out = _decompress_in_place(src, ops)
            if out is not None:
                return out if device else ops.to_numpy(out).reshape(out.shape)
        src = src.to_bytes()
    buf = memoryview(src).cast("B")
    h = parse_header(bytes(buf[:HEADER_SIZE]))
    if len(buf) != h.total_bytes:
        raise ArchiveFormatError(f"archive is {len(buf)} bytes, header promises {h.total_bytes}")
    dims = h.field_dims
    cfg = QuantConfig(eb=h.eb_resolved, cap=h.cap, block_shape=h.block_shape[: h.ndims])
    inner, n_global, cs = math.prod(dims[1:]), h.n_points, h.chunk_size
    if h.n_chunks != -(-n_global // cs):
        raise ArchiveFormatError(f"{h.n_chunks} chunks inconsistent with {n_global} points at "
                                 f"chunk size {cs}")
    rows = list(rows) if rows is not None else slab_rows(dims[0], cfg.block_shape[0], world)
    if len(rows) != world or sum(rows) != dims[0]:
        raise SdqzError("rows must give one slab height per rank covering axis 0")
    _check_rows(rows, cfg.block_shape[0])
    o, n_local = sum(rows[:rank]) * inner, rows[rank] * inner
    local_dims = (rows[rank],) + tuple(dims[1:])
    p = HEADER_SIZE
    bw = np.frombuffer(buf, np.uint8, h.cap, p)
    p += h.cap
    rec = np.frombuffer(buf, _RECORD, h.n_outliers, p)
    p += 16 * h.n_outliers
    bits = np.frombuffer(buf, "<u4", h.n_chunks, p)
    p += 4 * h.n_chunks
    offs = np.zeros(h.n_chunks + 1, np.int64)
    np.cumsum((bits.astype(np.int64) + 7) >> 3, out=offs[1:])
    if int(offs[-1]) != h.payload_bytes:
        raise ArchiveFormatError(f"payload of {h.payload_bytes} bytes disagrees with chunk bit "
                                 f"lengths ({int(offs[-1])} bytes)")
    idx = rec["index"]
    _validate_records(idx, n_global)
    if n_local == 0:
        return np.empty(local_dims, h.np_dtype)
    c0, c1 = o // cs, -(-(o + n_local) // cs)
    n_range = min(c1 * cs, n_global) - c0 * cs
    a, b = np.searchsorted(idx, o), np.searchsorted(idx, o + n_local)
    r = np.empty((max(b - a, 1), 2), np.uint64)
    r[: b - a, 0] = idx[a:b] - np.uint64(o)
    r[: b - a, 1] = rec["value"][a:b].view(np.uint64)
    pay = np.zeros(int(offs[c1] - offs[c0]) + 64, np.uint8)
    pay[: int(offs[c1] - offs[c0])] = np.frombuffer(buf, np.uint8, int(offs[c1] - offs[c0]), p + int(offs[c0]))
    out = ops.decompress_slab(h, ops.upload(bw.copy()), ops.upload(r.reshape(-1).view(np.int64)), int(b - a),
                              0, ops.upload(np.concatenate([bits[c0:c1], np.zeros(4, "<u4")]).view(np.int32))[:c1 - c0],
                              ops.upload(pay), int(offs[c1] - offs[c0]), n_range, o - c0 * cs, local_dims)
    return out if device else ops.to_numpy(out).reshape(local_dims)


def _decompress_in_place(ar: ShardedArchive, ops):
    """Each rank decodes its own chunks with its own records -- valid when
    every slab starts on a chunk boundary (then a rank's chunks cover exactly
    its slab); None otherwise (the caller falls back to the bytes path)."""
    import torch.distributed as dist
    h = ar.header
    rank = dist.get_rank(ar.group)
    dims = h.field_dims
    inner, cs = math.prod(dims[1:]), h.chunk_size
    offs = [sum(ar.rows[:r]) * inner for r in range(len(ar.rows) + 1)]
    if any(x % cs for x in offs[:-1]):
        return None
    o, n_local = offs[rank], offs[rank + 1] - offs[rank]
    local_dims = (ar.rows[rank],) + tuple(dims[1:])
    if n_local == 0:
        import torch
        return torch.empty(local_dims, dtype=torch.float32 if h.dtype_code == 0 else torch.float64,
                           device=ops.device)
    s = ar.sections
    k = int(ar.rank_sizes[rank, 2])
    n_range = min(-(-(o + n_local) // cs) * cs, h.n_points) - o
    return ops.decompress_slab(h, s["bitwidths"], s["outliers"], k, o, s["chunk_bits"], s["payload"],
                               s["payload_bytes"], n_range, 0, local_dims)


__all__ = ["DeviceShardOps", "ShardedArchive", "compress_sharded", "compress_sharded_device",
           "decompress_sharded", "slab_rows"]
