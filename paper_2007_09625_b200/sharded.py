"""Multi-GPU slab sharding of compress / decompress.

One process per GPU under `torch.distributed` (NCCL over NVLink on the box;
gloo in the CPU tests).  A field is split along axis 0 into slabs of whole
block-rows -- Lorenzo blocks are zero-padded and independent
(dualquant.py:81-86, :185-186), so every slab quantizes exactly as the same
rows of the whole field do.  Only global statistics and archive assembly are
exchanged:

  1. all-reduce of (min, max, nonfinite) -> identical resolved eb everywhere
     (core.py:161-175);
  2. per-slab dual-quant (K2) -> u16 codes + local u64 histogram;
  3. all-reduce SUM of the histogram -> every rank builds the identical
     codebook (K3 is deterministic);
  4. chunks of default_chunk_size(N_global) (huffman.py:206-212): a rank owns
     the chunks that START in its slab; the codes of a chunk straddling the
     slab end come from the following ranks' leading "head" codes (one
     all-gather of < chunk_size codes per rank);
  5. all-gather of the per-rank sections (outlier records with global
     indices, chunk bit lengths, payload); the archive is their concatenation
     in rank order, byte-identical to a single-GPU `compress` of the field.

`decompress_sharded` is the mirror: each rank inflates the chunk range that
covers its slab and reconstructs its rows with its outlier sub-range.

The per-rank compute goes through `DeviceShardOps` (libsdqz_cuda.so on this
rank's GPU).  The exchange protocol only sees torch tensors, so the CPU tests
drive it with a gloo group and a checker backend.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from .archive import HEADER_SIZE, ArchiveFormatError, ArchiveHeader, pack_header, parse_header
from .core import (ErrorBoundSpec, FieldDescriptor, QuantConfig, SdqzError, _as_dims,
                   resolve_error_bound)
from .huffman import default_chunk_size, select_unit_width

_RECORD = np.dtype([("index", "<u8"), ("value", "<f8")])


@dataclass
class Book:
    """A codebook as the shard backends exchange it."""

    bitwidths: np.ndarray     # uint8[cap]
    unit_width: int
    max_bitwidth: int
    handle: object = None     # backend-private (device tables)


# --------------------------------------------------------------------------
# per-rank compute on this rank's GPU
# --------------------------------------------------------------------------
class DeviceShardOps:
    """Stage calls of one rank through the C-ABI (include/sdqz_cuda.h)."""

    def __init__(self):
        _lib.require_cuda()

    @property
    def device(self):
        torch = _device._torch()
        return torch.device("cuda", torch.cuda.current_device())

    def field(self, local):
        return _device.to_device(_device.as_field(local))

    def describe(self, t, dt):
        return _device.describe(t, dt)

    def quantize(self, t, dt, local_dims, cfg: QuantConfig):
        """dualquant.py:242-273 on the slab -> (codes int16[n], hist int64[cap], nonfinite)."""
        from .dualquant import _codes_device
        n = math.prod(local_dims)
        codes, hist, nonfinite = _codes_device(t, 0 if dt == np.float32 else 1, local_dims, cfg, True)
        return codes[:n], hist, nonfinite

    def codebook(self, hist, cap: int) -> Book:
        """build_tree + canonize (huffman.py:98-190) on the device."""
        from .huffman import _canonize_device
        torch = _device._torch()
        bw = _device.empty(cap + 16, torch.uint8)
        ctx = _lib.context()
        ctx.call("sdqz_build_tree", _lib.ptr(hist), cap, _lib.ptr(bw))
        ent, first, offs, syms, unit, mx, _ = _canonize_device(bw, cap)
        return Book(_device.download(bw, cap).copy(), unit, mx, (ent, first, offs, syms, bw))

    def deflate(self, codes, chunk: int, book: Book, cap: int):
        """encode + deflate (huffman.py:193-269) -> (chunk_bits int32 tensor, payload uint8 tensor)."""
        torch = _device._torch()
        n = codes.numel()
        nch = -(-n // chunk) if n else 0
        bits = _device.empty(nch, torch.int32)
        if n == 0:
            return bits[:0], _device.empty(0, torch.uint8)[:0]
        cap_bytes = -(-n * book.max_bitwidth // 8) + nch + 64
        pay = _device.empty(cap_bytes, torch.uint8)
        pb = _lib.c_uint64()
        codes = codes.contiguous()
        _lib.context().call("sdqz_encode_deflate", _lib.ptr(codes), n, _lib.ptr(book.handle[0]),
                            cap, int(chunk), _lib.ptr(bits), _lib.ptr(pay), cap_bytes,
                            _lib.byref(pb))
        return bits[:nch], pay[: pb.value]

    def outliers(self, t, dt, codes, eb: float):
        """Ordered outlier list of the slab (dualquant.py:190-194) as an int64 tensor of
        {index, f64 bits} pairs with slab-local indices."""
        torch = _device._torch()
        n = codes.numel()
        rec = _device.empty(2 * n + 2, torch.int64)
        k = _lib.c_uint64()
        _lib.context().call("sdqz_outliers", _lib.ptr(t), 0 if dt == np.float32 else 1,
                            _lib.ptr(codes), n, float(eb), _lib.ptr(rec), n + 1, _lib.byref(k))
        return rec[: 2 * k.value]

    def inflate(self, payload: np.ndarray, chunk_bits: np.ndarray, chunk: int, n_codes: int,
                bitwidths: np.ndarray):
        """Chunk-range inflate (huffman.py:311-356) -> uint32 codes (host)."""
        from .huffman import DeflatedStream, canonize, inflate
        _, rb = canonize(bitwidths)
        return inflate(DeflatedStream(chunk, chunk_bits, payload.tobytes()), rb, n_codes)

    def decompress_slab(self, h: ArchiveHeader, bw: np.ndarray, rec: np.ndarray, bits: np.ndarray,
                        payload: np.ndarray, n_range: int, lo: int, local_dims) -> np.ndarray:
        """Device-resident slab decompress (sdqz_decompress_slab): the chunk range's
        sections go to the GPU once; decode tables, the warp-parallel decoder and
        the reconstruct run there, and only the slab comes back."""
        torch = _device._torch()
        ch = _lib.Header()
        ch.dtype_code, ch.ndims, ch.eb_mode, ch.unit_width = h.dtype_code, h.ndims, h.eb_mode, h.unit_width
        for a in range(3):
            ch.dims[a] = h.dims[a]
            ch.block[a] = h.block_shape[a]
        ch.eb_resolved, ch.eb_specified, ch.cap, ch.chunk_size = (h.eb_resolved, h.eb_specified, h.cap,
                                                                  h.chunk_size)
        ch.n_outliers, ch.n_chunks, ch.payload_bytes = len(rec), len(bits), len(payload)
        bwp = np.zeros(h.cap + 16, np.uint8)
        bwp[: h.cap] = bw
        r = np.empty((max(len(rec), 1), 2), np.uint64)
        r[: len(rec), 0] = rec["index"]
        r[: len(rec), 1] = rec["value"].view(np.uint64)
        pay = np.zeros(len(payload) + 64, np.uint8)
        pay[: len(payload)] = payload
        d_bw = _device.upload(bwp)
        d_rec = _device.upload(r.reshape(-1).view(np.int64))
        d_bits = _device.upload(np.concatenate([bits.astype(np.uint32), np.zeros(4, np.uint32)]).view(np.int32))
        d_pay = _device.upload(pay)
        n = math.prod(local_dims)
        out = _device.empty(n, torch.float32 if h.dtype_code == 0 else torch.float64)
        _lib.context().call("sdqz_decompress_slab", ctypes.byref(ch), _lib.ptr(d_bw), _lib.ptr(d_rec),
                            len(rec), _lib.ptr(d_bits), len(bits), _lib.ptr(d_pay), len(payload),
                            int(n_range), int(lo), _lib.dims3(local_dims), _lib.ptr(out))
        return _device.download(out, n).reshape(local_dims)

    def reconstruct(self, codes: np.ndarray, idx: np.ndarray, vals: np.ndarray, local_dims,
                    cfg: QuantConfig, dtype) -> np.ndarray:
        """reconstruct_field (dualquant.py:299-332) + astype (pipeline.py:53) of the slab."""
        torch = _device._torch()
        n = math.prod(local_dims)
        c32 = _device.upload(np.ascontiguousarray(codes, dtype=np.uint32).view(np.int32))
        di = _device.upload(idx.astype(np.uint64).view(np.int64)) if idx.size else None
        dv = _device.upload(vals.astype(np.float64)) if idx.size else None
        f32 = np.dtype(dtype) == np.float32
        out = _device.empty(n, torch.float32 if f32 else torch.float64)
        _lib.context().call("sdqz_reconstruct", _lib.ptr(c32), 4, n, _lib.ptr(di), _lib.ptr(dv),
                            int(idx.size), len(local_dims), _lib.dims3(local_dims),
                            _lib.block3(cfg.block_shape), float(cfg.eb), int(cfg.cap),
                            _lib.ptr(out), 0 if f32 else 1)
        return _device.download(out, n).reshape(local_dims)


# --------------------------------------------------------------------------
# collectives (tensors live on the group's device: CUDA for NCCL, CPU for gloo)
# --------------------------------------------------------------------------
def _comm_device(group):
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _allgather_i64(values, group):
    import torch
    import torch.distributed as dist
    dev = _comm_device(group)
    world = dist.get_world_size(group)
    t = torch.tensor(list(values), dtype=torch.int64, device=dev)
    out = torch.empty(world * t.numel(), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(out, t, group=group)
    return out.view(world, -1).cpu().numpy()


def _allgather_bytes(t, group):
    """Variable-length uint8 tensors -> list of per-rank uint8 tensors (comm device)."""
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


# --------------------------------------------------------------------------
# compress
# --------------------------------------------------------------------------
def compress_sharded(local, dims, *, eb: float, mode: str = "abs", cap: int = 1024,
                     block_shape=None, chunk_size: int | None = None, group=None,
                     ops=None) -> bytes:
    """Compress a field whose axis-0 slabs are spread over the ranks of `group`.

    `local` is this rank's slab (rows of the global field, in rank order);
    `dims` the GLOBAL dims.  Every rank returns the archive bytes, identical to
    `compress(whole_field, dims, ...)` on one GPU (pipeline.py:15-39)."""
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
    spec = ErrorBoundSpec(mode, eb)
    probe = QuantConfig.for_rank(1.0, nd, cap=cap, block_shape=block_shape)
    b0 = probe.block_shape[0]
    for i, r in enumerate(rows[:-1]):
        if r % b0:
            raise SdqzError(f"slab {i} has {r} rows; every slab but the last must be a "
                            f"multiple of the block extent {b0}")
    o = sum(rows[:rank]) * inner

    # 1. global range -> eb (core.py:136-175)
    if n_local:
        vmin, vmax, nonfinite = ops.describe(t, dt)
    else:
        vmin, vmax, nonfinite = math.inf, -math.inf, False
    dev = _comm_device(group)
    st = torch.tensor([-vmin, vmax, 1.0 if nonfinite else 0.0], dtype=torch.float64, device=dev)
    dist.all_reduce(st, op=dist.ReduceOp.MAX, group=group)
    gmin, gmax, gnf = -float(st[0]), float(st[1]), bool(st[2] > 0)
    fd = FieldDescriptor(dims, n_global, gmin, gmax, gnf, np.dtype(dt))
    ebr = resolve_error_bound(spec, fd)
    cfg = QuantConfig.for_rank(ebr, nd, cap=cap, block_shape=block_shape)
    if chunk_size is not None and chunk_size < 1:
        raise SdqzError("chunk_size must be >= 1")
    cs = int(chunk_size or default_chunk_size(n_global))

    # 2. slab dual-quant + 3. global histogram -> identical codebook
    local_dims = (rows_local,) + dims[1:]
    if n_local:
        codes, hist, _ = ops.quantize(t, dt, local_dims, cfg)
    else:
        codes = torch.empty(0, dtype=torch.int16, device=ops.device)
        hist = torch.zeros(cap, dtype=torch.int64, device=ops.device)
    h = hist.to(dev)
    dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
    book = ops.codebook(h.to(ops.device), cap)

    # 4. chunk ownership + head exchange
    first_own = min(-(-o // cs) * cs, o + n_local)     # first chunk start inside the slab
    head = codes[: first_own - o]
    heads = _allgather_bytes(_as_bytes(head), group)
    own = codes[first_own - o:]
    if first_own < o + n_local:
        end = min(-(-(o + n_local) // cs) * cs, n_global)
        need = end - (o + n_local)
        tails = []
        for r in range(rank + 1, world):
            if need <= 0:
                break
            hr = heads[r].view(torch.int16)
            take = min(need, hr.numel())
            tails.append(hr[:take].to(ops.device))
            need -= take
        if need:
            raise SdqzError("internal: straddling chunk not covered by the following slabs")
        if tails:
            own = torch.cat([own] + tails)
    bits, payload = ops.deflate(own, cs, book, cap)

    # outliers with global indices (ascending: slabs are in rank order)
    rec = ops.outliers(t, dt, codes, cfg.eb) if n_local else \
        torch.empty(0, dtype=torch.int64, device=ops.device)
    if rec.numel():
        rec = rec.view(-1, 2).clone()
        rec[:, 0] += o
    # 5. assembly: all ranks gather every section
    g_rec = _allgather_bytes(_as_bytes(rec), group)
    g_bits = _allgather_bytes(_as_bytes(bits), group)
    g_pay = _allgather_bytes(_as_bytes(payload), group)
    n_out = sum(x.numel() for x in g_rec) // 16
    n_chunks = sum(x.numel() for x in g_bits) // 4
    p_bytes = sum(x.numel() for x in g_pay)
    if n_chunks != -(-n_global // cs):
        raise SdqzError("internal: chunk count mismatch after assembly")
    hdr = ArchiveHeader(
        dtype_code=0 if dt == np.float32 else 1, ndims=nd, eb_mode=0 if mode == "abs" else 1,
        dims=tuple(dims) + (1,) * (3 - nd), eb_resolved=cfg.eb, eb_specified=float(eb), cap=cap,
        block_shape=tuple(cfg.block_shape) + (1,) * (3 - nd), chunk_size=cs,
        unit_width=select_unit_width(book.max_bitwidth), n_outliers=n_out, n_chunks=n_chunks,
        payload_bytes=p_bytes)
    body = torch.cat([x.cpu() for x in g_rec + g_bits + g_pay]) if n_global else None
    parts = [pack_header(hdr), np.ascontiguousarray(book.bitwidths, dtype=np.uint8).tobytes()]
    if body is not None:
        parts.append(body.numpy().tobytes())
    return b"".join(parts)


# --------------------------------------------------------------------------
# decompress
# --------------------------------------------------------------------------
def decompress_sharded(blob, *, group=None, rows: list[int] | None = None, ops=None) -> np.ndarray:
    """Reconstruct this rank's slab of the archive's field (pipeline.py:42-58 on a
    row range).  `rows` gives every rank's slab height (default: an even split
    in whole block-rows).  Returns the slab shaped (rows_r, *dims[1:])."""
    import torch.distributed as dist

    ops = ops or DeviceShardOps()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    buf = memoryview(blob).cast("B")
    h = parse_header(bytes(buf[:HEADER_SIZE]))
    if len(buf) != h.total_bytes:
        raise ArchiveFormatError(f"archive is {len(buf)} bytes, header promises {h.total_bytes}")
    dims = h.field_dims
    cfg = QuantConfig(eb=h.eb_resolved, cap=h.cap, block_shape=h.block_shape[: h.ndims])
    inner, n_global, cs = math.prod(dims[1:]), h.n_points, h.chunk_size
    if h.n_chunks != -(-n_global // cs):
        raise ArchiveFormatError(f"{h.n_chunks} chunks inconsistent with {n_global} points at "
                                 f"chunk size {cs}")
    rows = rows or slab_rows(dims[0], cfg.block_shape[0], world)
    if len(rows) != world or sum(rows) != dims[0]:
        raise SdqzError("rows must give one slab height per rank covering axis 0")
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
    if n_local == 0:
        return np.empty(local_dims, h.np_dtype)
    c0, c1 = o // cs, -(-(o + n_local) // cs)
    payload = np.frombuffer(buf, np.uint8, int(offs[c1] - offs[c0]), p + int(offs[c0]))
    n_range = min(c1 * cs, n_global) - c0 * cs
    lo = o - c0 * cs
    idx = rec["index"]
    a, b = np.searchsorted(idx, o), np.searchsorted(idx, o + n_local)
    if hasattr(ops, "decompress_slab"):   # device backend: one device-resident pass
        srec = np.empty(b - a, _RECORD)
        srec["index"] = idx[a:b] - np.uint64(o)
        srec["value"] = rec["value"][a:b]
        return ops.decompress_slab(h, bw.copy(), srec, bits[c0:c1].copy(), payload, n_range, lo, local_dims)
    codes = ops.inflate(payload, bits[c0:c1].copy(), cs, n_range, bw.copy())
    codes = np.asarray(codes)[lo: lo + n_local]
    return ops.reconstruct(codes, (idx[a:b] - np.uint64(o)).astype(np.uint64),
                           rec["value"][a:b].astype(np.float64), local_dims, cfg, h.np_dtype)


__all__ = ["Book", "DeviceShardOps", "compress_sharded", "decompress_sharded", "slab_rows"]
