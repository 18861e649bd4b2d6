"""End-to-end compress / decompress (reference: sdqz/pipeline.py:15-58).

The drop-in entry points keep the reference's signatures.  Behind them one
fused C-ABI call runs the whole device pipeline:

  compress:   describe (valrel) -> resolve eb -> dual-quant + histogram ->
              tree + canonical codebook -> chunk bit counts -> offset scan ->
              pack payload + compact outliers           (all on the GPU)
  decompress: canonical tables + LUT -> inflate -> outlier scatter / checks ->
              reconstruct                               (all on the GPU)

Host work is O(1) validation, the 93-byte header, and the host<->device
copies of the input field / archive bytes.  `compress_device` /
`decompress_device` are the same pipelines with device-resident inputs and
outputs (the bench's kernel-level figure).
"""

from __future__ import annotations

import ctypes
import math
import struct
from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from .archive import Archive, ArchiveFormatError
from .core import (DEFAULT_BLOCK_SHAPES, ErrorBoundSpec, QuantConfig, SdqzError, _as_dims)

_PyBytes_FromStringAndSize = ctypes.pythonapi.PyBytes_FromStringAndSize
_PyBytes_FromStringAndSize.restype = ctypes.py_object
_PyBytes_FromStringAndSize.argtypes = [ctypes.c_void_p, ctypes.c_ssize_t]
_PyBytes_AsString = ctypes.pythonapi.PyBytes_AsString
_PyBytes_AsString.restype = ctypes.c_void_p
_PyBytes_AsString.argtypes = [ctypes.py_object]


@dataclass
class DeviceArchive:
    """Archive sections resident in a context's device memory.

    The sections live in the context's scratch arena until the next compress
    on that context; `gen` identifies this archive, and the C-ABI refuses a
    stale handle (SdqzError) instead of handing out the newer archive."""

    header: _lib.Header
    ctx: _lib.Context
    gen: int = 0

    @property
    def nbytes(self) -> int:
        return self.header.total_bytes

    @property
    def valid(self) -> bool:
        return self.gen != 0 and self.ctx.archive_generation == self.gen

    def to_bytes(self) -> bytes:
        n = self.header.total_bytes
        out = _PyBytes_FromStringAndSize(None, n)
        self.ctx.call("sdqz_archive_write", self.gen, ctypes.c_void_p(_PyBytes_AsString(out)), n)
        return out

    def write_into(self, host_ptr: int, capacity: int) -> int:
        self.ctx.call("sdqz_archive_write", self.gen, ctypes.c_void_p(host_ptr), capacity)
        return self.header.total_bytes

    def sections(self):
        """Device pointers (bitwidths, outlier records, chunk bits, payload)."""
        ptrs = [ctypes.c_void_p() for _ in range(4)]
        self.ctx.call("sdqz_archive_sections", self.gen, *(ctypes.byref(p) for p in ptrs))
        return ptrs


def _check_request(arr, dims, eb, mode, cap, block_shape, chunk_size):
    """Host-side checks in the reference's order; returns (dims, block, pending
    error) where the pending error is one the reference raises only after
    resolve_error_bound (QuantConfig / deflate checks)."""
    if dims is None:
        shape = tuple(arr.shape)
        dims = shape if len(shape) > 1 else (_device.numel(arr),)
    dims = _as_dims(dims)
    n = math.prod(dims)
    if _device.numel(arr) != n:
        raise SdqzError(f"data has {_device.numel(arr)} values but dims {'x'.join(map(str, dims))} "
                        f"require {n}")
    if len(dims) > 3:
        raise SdqzError(f"rank {len(dims)} fields are not supported (1-3)")
    ErrorBoundSpec(mode, eb)
    pending = None
    block = None
    try:
        # QuantConfig with a stand-in bound: validates block rank, cap, extents
        block = QuantConfig.for_rank(1.0, len(dims), cap=cap, block_shape=block_shape).block_shape
    except SdqzError as e:
        pending = e
    if pending is None and chunk_size is not None and chunk_size != 0 and chunk_size < 1:
        pending = SdqzError("chunk_size must be >= 1")
    if pending is None and chunk_size is not None and chunk_size > 0xFFFFFFFF:
        # the header stores chunk_size as u32 (archive.py:34-35): the reference's
        # serialize fails in struct.pack; never truncate it into another archive
        pending = struct.error("'I' format requires 0 <= number <= 4294967295")
    return dims, block, pending


def _raise_resolve_errors(t, dt, mode, eb):
    """Run the device describe and raise what resolve_error_bound /
    QuantConfig would raise first (core.py:161-175, :87-89)."""
    from .core import FieldDescriptor, resolve_error_bound
    vmin, vmax, nonfinite = _device.describe(t, dt)
    fd = FieldDescriptor((t.numel(),), t.numel(), vmin, vmax, nonfinite, dt)
    ebr = resolve_error_bound(ErrorBoundSpec(mode, eb), fd)
    if not (ebr > 0 and math.isfinite(ebr)):
        raise SdqzError("error bound must be positive and finite")


def compress_device(data, dims=None, *, eb: float, mode: str = "abs", cap: int = 1024,
                    block_shape=None, chunk_size: int | None = None, stats=None) -> DeviceArchive:
    """compress() whose input may be a CUDA tensor and whose output stays on
    the device (sections in the calling thread's context).  `stats` =
    (vmin, vmax, nonfinite) of an earlier describe of the same unchanged
    field skips the describe pass (sdqz_compress_described; rd_sweep)."""
    arr = _device.as_field(data)
    dims, block, pending = _check_request(arr, dims, eb, mode, cap, block_shape, chunk_size)
    t, dt = _device.to_device(arr)
    if pending is not None:
        _raise_resolve_errors(t, dt, mode, eb)
        raise pending
    ctx = _lib.context()
    hdr = _lib.Header()
    args = (_lib.ptr(t), 0 if dt == np.float32 else 1, len(dims), _lib.dims3(dims), _lib.block3(block),
            0 if mode == "abs" else 1, float(eb), int(cap), int(chunk_size or 0))
    if stats is None:
        ctx.call("sdqz_compress", *args, ctypes.byref(hdr))
    else:
        ctx.call("sdqz_compress_described", *args,
                 (ctypes.c_double * 3)(float(stats[0]), float(stats[1]), 1.0 if stats[2] else 0.0),
                 ctypes.byref(hdr))
    return DeviceArchive(hdr, ctx, ctx.archive_generation)


def compress(data, dims=None, *, eb: float, mode: str = "abs", cap: int = 1024,
             block_shape: tuple[int, ...] | None = None, chunk_size: int | None = None,
             workers: int | None = None) -> bytes:
    """Compress a 1-3D float field into archive bytes (pipeline.py:15-39).

    `workers` is accepted for API compatibility and never changes the bytes."""
    return compress_device(data, dims, eb=eb, mode=mode, cap=cap, block_shape=block_shape,
                           chunk_size=chunk_size).to_bytes()


def compress_host(data, dims=None, *, eb: float, mode: str = "abs", cap: int = 1024,
                  block_shape=None, chunk_size: int | None = None) -> bytes:
    """compress() of a host array through the host-buffer C-ABI
    (sdqz_compress_host): the field is staged to the device by the library,
    the archive comes back the same way; torch is never imported."""
    arr = np.asarray(data)
    dims, block, pending = _check_request(arr, dims, eb, mode, cap, block_shape, chunk_size)
    dt = _device.field_dtype(arr)
    a = np.ascontiguousarray(arr, dtype=dt).reshape(-1)
    if pending is not None:
        # what resolve_error_bound raises first (core.py:161-175), then the pending error
        from .core import describe_field, resolve_error_bound
        ebr = resolve_error_bound(ErrorBoundSpec(mode, eb), describe_field(a, (a.size,)))
        if not (ebr > 0 and math.isfinite(ebr)):
            raise SdqzError("error bound must be positive and finite")
        raise pending
    ctx = _lib.host_context()
    hdr = _lib.Header()
    ctx.call("sdqz_compress_host", ctypes.c_void_p(a.ctypes.data), 0 if dt == np.float32 else 1,
             len(dims), _lib.dims3(dims), _lib.block3(block), 0 if mode == "abs" else 1, float(eb),
             int(cap), int(chunk_size or 0), ctypes.byref(hdr))
    n = hdr.total_bytes
    out = _PyBytes_FromStringAndSize(None, n)
    ctx.call("sdqz_archive_write", ctx.archive_generation, ctypes.c_void_p(_PyBytes_AsString(out)), n)
    return out


def decompress_host(blob: bytes) -> np.ndarray:
    """decompress() into a host array through the host-buffer C-ABI
    (sdqz_decompress_host); torch is never imported."""
    blob = bytes(blob)
    ctx = _lib.host_context()
    h = _lib.Header()
    base = ctypes.c_void_p(_PyBytes_AsString(blob))
    try:
        ctx.call("sdqz_parse_header", base, len(blob), ctypes.byref(h))
    except ArchiveFormatError as e:
        if str(e) == "bad magic":
            raise ArchiveFormatError(f"bad magic {blob[:4]!r}") from None
        raise
    dims = _dims_of(h)
    out = np.empty(math.prod(dims), np.float32 if h.dtype_code == 0 else np.float64)
    try:
        ctx.call("sdqz_decompress_host", base, len(blob), ctypes.c_void_p(out.ctypes.data))
        _check_geometry(h)
    except SdqzError as e:
        _rewrite_geometry_error(e, blob)
        raise
    return out.reshape(dims)


def _dims_of(h) -> tuple[int, ...]:
    return tuple(int(h.dims[a]) for a in range(h.ndims))


def _out_tensor(h, out=None):
    torch = _device._torch()
    n = math.prod(_dims_of(h))
    tdt = torch.float32 if h.dtype_code == 0 else torch.float64
    if out is not None:
        if out.numel() != n or out.dtype != tdt or not out.is_cuda or not out.is_contiguous():
            raise SdqzError("out tensor does not match the archive")
        return out
    return _device.empty(n, tdt)


def decompress_device(src, out=None):
    """Decompress to a CUDA tensor.  `src` is a DeviceArchive (sections
    already on the device) or archive bytes (copied host -> device)."""
    if isinstance(src, DeviceArchive):
        ctx = src.ctx
        ctx.sync_stream()
        h = src.header
        bw, rec, cb, pay = src.sections()
        o = _out_tensor(h, out)
        ctx.call("sdqz_decompress_sections", ctypes.byref(h), bw, rec, cb, pay, _lib.ptr(o))
        return o.view(*_dims_of(h))
    blob = bytes(src) if not isinstance(src, (bytes, bytearray, memoryview)) else src
    ctx = _lib.context()
    h = _lib.Header()
    mv = memoryview(blob).cast("B")
    buf = (ctypes.c_char * len(mv)).from_buffer_copy(mv) if not isinstance(blob, bytes) else None
    base = ctypes.c_void_p(_PyBytes_AsString(blob)) if isinstance(blob, bytes) else \
        ctypes.cast(buf, ctypes.c_void_p)
    try:
        ctx.call("sdqz_parse_header", base, len(mv), ctypes.byref(h))
    except ArchiveFormatError as e:
        if str(e) == "bad magic":
            raise ArchiveFormatError(f"bad magic {bytes(mv[:4])!r}") from None
        raise
    o = _out_tensor(h, out)
    ctx.call("sdqz_decompress", base, len(mv), _lib.ptr(o))
    _check_geometry(h)
    return o.view(*_dims_of(h))


def decompress_quality(src: DeviceArchive, orig, out=None):
    """decompress_device(src) and the quality sums of the result against
    `orig` in one pass: the reduction runs in the reconstruct kernels'
    epilogue (sdqz_decompress_quality).  Returns (field, q5, fused) with q5 =
    (sum d^2, max |d|, min orig, max orig, nonfinite(orig)) -- metrics.quality's
    inputs -- and fused False when this path scored in a separate pass."""
    ctx = src.ctx
    ctx.sync_stream()
    h = src.header
    bw, rec, cb, pay = src.sections()
    o = _out_tensor(h, out)
    t, dt = _device.to_device(_device.as_field(orig))
    if t.numel() != o.numel():
        raise SdqzError(f"length mismatch: {t.numel()} vs {o.numel()} values")
    q5 = (ctypes.c_double * 5)()
    fused = ctypes.c_int(0)
    ctx.call("sdqz_decompress_quality", ctypes.byref(h), bw, rec, cb, pay, _lib.ptr(o), _lib.ptr(t),
             0 if dt == np.float32 else 1, q5, ctypes.byref(fused))
    return o.view(*_dims_of(h)), tuple(q5), bool(fused.value)


def _check_geometry(h):
    block = tuple(int(h.block[a]) for a in range(h.ndims))
    QuantConfig(eb=h.eb_resolved, cap=h.cap, block_shape=block)


def decompress(blob: bytes, workers: int | None = None) -> np.ndarray:
    """Parse archive bytes and reconstruct the field (pipeline.py:56-58):
    shaped, in the archive dtype."""
    try:
        t = decompress_device(blob)
    except SdqzError as e:
        _rewrite_geometry_error(e, blob)
        raise
    return _device.download(t)


def _rewrite_geometry_error(e, blob):
    msg = str(e)
    if msg == "all extents must be >= 1" and len(blob) >= 93:
        from .archive import parse_header
        h = parse_header(blob)
        raise SdqzError(f"all extents must be >= 1, got {h.block_shape[:h.ndims]}") from None


def decompress_archive(ar: Archive, workers: int | None = None) -> np.ndarray:
    """Reconstruct a parsed archive (pipeline.py:42-53)."""
    h = ar.header
    QuantConfig(eb=h.eb_resolved, cap=h.cap, block_shape=h.block_shape[:h.ndims])
    torch = _device._torch()
    ch = _lib.Header()
    ch.dtype_code, ch.ndims, ch.eb_mode, ch.unit_width = h.dtype_code, h.ndims, h.eb_mode, h.unit_width
    for a in range(3):
        ch.dims[a] = h.dims[a]
        ch.block[a] = h.block_shape[a]
    ch.eb_resolved, ch.eb_specified, ch.cap, ch.chunk_size = (h.eb_resolved, h.eb_specified,
                                                              h.cap, h.chunk_size)
    k = int(np.asarray(ar.outlier_indices).size)
    ch.n_outliers = k
    ch.n_chunks = int(np.asarray(ar.chunk_bit_lengths).size)
    ch.payload_bytes = len(ar.payload)
    bw = np.zeros(h.cap + 16, np.uint8)
    bw[: h.cap] = np.asarray(ar.bitwidths, dtype=np.uint8)[: h.cap]
    rec = np.empty((max(k, 1), 2), np.uint64)
    rec[:k, 0] = np.asarray(ar.outlier_indices, dtype=np.uint64)
    rec[:k, 1] = np.asarray(ar.outlier_values, dtype=np.float64).view(np.uint64)
    pay = np.zeros(len(ar.payload) + 64, np.uint8)
    pay[: len(ar.payload)] = np.frombuffer(ar.payload, np.uint8)
    cb = np.asarray(ar.chunk_bit_lengths, dtype=np.uint32)
    d_bw = _device.upload(bw)
    d_rec = _device.upload(rec.reshape(-1).view(np.int64))
    d_cb = _device.upload(np.concatenate([cb, np.zeros(4, np.uint32)]).view(np.int32))
    d_pay = _device.upload(pay)
    o = _out_tensor(ch)
    _lib.context().call("sdqz_decompress_sections", ctypes.byref(ch), _lib.ptr(d_bw),
                        _lib.ptr(d_rec), _lib.ptr(d_cb), _lib.ptr(d_pay), _lib.ptr(o))
    del torch
    return _device.download(o.view(*_dims_of(ch)))


__all__ = ["compress", "decompress", "decompress_archive", "compress_device",
           "decompress_device", "compress_host", "decompress_host", "decompress_quality", "DeviceArchive",
           "DEFAULT_BLOCK_SHAPES"]


class CompressPlan:
    """Pre-validated compress of one device-resident field: `run()` is a single
    C-ABI call (no per-call Python validation) -- used by the bench's
    device-level figure and by repeated compression of a resident field."""

    def __init__(self, t, dims, *, eb, mode="abs", cap=1024, block_shape=None, chunk_size=None):
        dims, block, pending = _check_request(t, dims, eb, mode, cap, block_shape, chunk_size)
        if pending is not None:
            raise pending
        self.t, dt = _device.to_device(t)
        self.ctx = _lib.context()
        self.args = (_lib.ptr(self.t), 0 if dt == np.float32 else 1, len(dims), _lib.dims3(dims),
                     _lib.block3(block), 0 if mode == "abs" else 1, float(eb), int(cap),
                     int(chunk_size or 0))
        self.hdr = _lib.Header()

    def run(self) -> DeviceArchive:
        self.ctx.call("sdqz_compress", *self.args, ctypes.byref(self.hdr))
        return DeviceArchive(self.hdr.copy(), self.ctx, self.ctx.archive_generation)


class DecompressPlan:
    """Device-resident decompress of the context's last archive into a
    preallocated output tensor (single C-ABI call per run)."""

    def __init__(self, dev: DeviceArchive):
        self.dev = dev
        self.out = _out_tensor(dev.header)

    def run(self, dev: DeviceArchive | None = None):
        """Decompress `dev` (default: the plan's archive) into the plan's buffer."""
        dev = dev or self.dev
        ctx, h = dev.ctx, dev.header
        bw, rec, cb, pay = dev.sections()
        ctx.call("sdqz_decompress_sections", ctypes.byref(h), bw, rec, cb, pay, _lib.ptr(self.out))
        return self.out
