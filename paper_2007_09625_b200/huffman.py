"""Lossless stage: canonical Huffman over quantization codes.

API mirror of the reference's huffman module (sdqz/huffman.py): the same
dataclasses, unit layout (bitwidth in the top 8 bits of a 32/64-bit unit),
byte-aligned MSB-first chunks and error messages.  Histogram, tree,
canonical codebook, encode, deflate and inflate execute on the GPU
(csrc/huffman.cu); only O(1) parameter logic stays on the host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from .core import CorruptionError, SdqzError
from .dualquant import CODE_DTYPE

WIDTH_FIELD_BITS = 8
MAX_CODEWORD_BITS = 64 - WIDTH_FIELD_BITS


@dataclass
class Codebook:
    """Forward table: one packed bitwidth+codeword unit per symbol (huffman.py:32-50)."""

    entries: np.ndarray
    unit_width: int

    @property
    def cap(self) -> int:
        return int(self.entries.size)

    @property
    def bitwidths(self) -> np.ndarray:
        return (self.entries >> np.uint64(self.unit_width - WIDTH_FIELD_BITS)).astype(np.uint8)

    @property
    def codewords(self) -> np.ndarray:
        mask = np.uint64((1 << (self.unit_width - WIDTH_FIELD_BITS)) - 1)
        return self.entries.astype(np.uint64) & mask


@dataclass
class ReverseCodebook:
    """Canonical decode tables (huffman.py:53-65)."""

    first_codes: np.ndarray  # uint64, index = bitwidth
    offsets: np.ndarray      # int64, one-past-end sentinel
    symbols: np.ndarray      # uint32, sorted by (bitwidth, symbol)
    max_bitwidth: int


@dataclass
class DeflatedStream:
    """Byte-aligned chunks of MSB-first concatenated codewords (huffman.py:68-74)."""

    chunk_size: int
    chunk_bit_lengths: np.ndarray  # uint32
    payload: bytes


def _pow2_at_least(n: int, lo: int = 4) -> int:
    p = lo
    while p < n:
        p <<= 1
    return p


def _check_codes(codes: np.ndarray, cap: int) -> None:
    """Host-side guard only for inputs a uint32 upload could alias (wide or signed)."""
    if codes.size and (codes.dtype.itemsize > 4 or codes.dtype.kind == "i"):
        if int(codes.min()) < 0 or int(codes.max()) >= cap:
            raise CorruptionError(f"quantization code outside [0, {cap})")


def histogram(codes, cap: int, workers: int | None = None) -> np.ndarray:
    """Exact frequency of each code; code >= cap is corruption (huffman.py:77-95)."""
    codes = np.asarray(codes).reshape(-1)
    if codes.size == 0:
        return np.zeros(cap, dtype=np.int64)
    _check_codes(codes, cap)
    torch = _device._torch()
    d = _device.upload(codes.astype(np.uint32, copy=False).view(np.int32))
    h = _device.empty(cap, torch.int64)
    _lib.context().call("sdqz_histogram_u32", _lib.ptr(d), codes.size, int(cap), _lib.ptr(h))
    return _device.download(h, cap).astype(np.int64)


def build_tree(freq) -> np.ndarray:
    """Optimal prefix-code bitwidths; ties break on (weight, smallest symbol)
    (huffman.py:98-131).  Runs the device two-queue merge."""
    f = np.asarray(freq, dtype=np.int64).reshape(-1)
    if f.size > 65536:
        raise SdqzError("histograms wider than 65536 symbols are not supported")
    cap = _pow2_at_least(f.size)
    padded = np.zeros(cap, dtype=np.int64)
    padded[: f.size] = np.maximum(f, 0)
    torch = _device._torch()
    dh = _device.upload(padded)
    bw = _device.empty(cap + 16, torch.uint8)
    _lib.context().call("sdqz_build_tree", _lib.ptr(dh), cap, _lib.ptr(bw))
    return _device.download(bw, f.size).astype(np.uint8)


def select_unit_width(max_bitwidth: int) -> int:
    """32-bit units when every codeword fits, 64-bit otherwise (huffman.py:134-143)."""
    if max_bitwidth < 1:
        raise SdqzError("maximum bitwidth must be >= 1")
    if max_bitwidth > MAX_CODEWORD_BITS:
        raise SdqzError(f"codeword bitwidth {max_bitwidth} exceeds the supported maximum "
                        f"of {MAX_CODEWORD_BITS}")
    return 32 if max_bitwidth <= 32 - WIDTH_FIELD_BITS else 64


def _canonize_device(bw_dev, cap: int):
    torch = _device._torch()
    ent = _device.empty(cap, torch.int64)
    first = _device.empty(64, torch.int64)
    offs = _device.empty(64, torch.int64)
    syms = _device.empty(cap, torch.int32)
    unit, mx, npres = _lib.c_int(), _lib.c_int(), _lib.c_uint32()
    _lib.context().call("sdqz_canonize", _lib.ptr(bw_dev), cap, _lib.ptr(ent), _lib.ptr(first),
                        _lib.ptr(offs), _lib.ptr(syms), _lib.byref(unit), _lib.byref(mx),
                        _lib.byref(npres))
    return ent, first, offs, syms, unit.value, mx.value, npres.value


def canonize(bitwidths) -> tuple[Codebook, ReverseCodebook]:
    """Canonical codewords for the given bitwidths (huffman.py:146-190)."""
    bw = np.asarray(bitwidths, dtype=np.uint8).reshape(-1)
    if bw.size > 65536:
        raise SdqzError("codebooks wider than 65536 symbols are not supported")
    cap = _pow2_at_least(bw.size)
    padded = np.zeros(cap + 16, dtype=np.uint8)
    padded[: bw.size] = bw
    ent, first, offs, syms, unit, mx, npres = _canonize_device(_device.upload(padded), cap)
    entries = _device.download(ent, bw.size).view(np.uint64)
    entries = entries.astype(np.uint32) if unit == 32 else entries.copy()
    rb = ReverseCodebook(first_codes=_device.download(first, mx + 1).view(np.uint64).copy(),
                         offsets=_device.download(offs, mx + 2).astype(np.int64),
                         symbols=_device.download(syms, npres).view(np.uint32).copy(),
                         max_bitwidth=int(mx))
    return Codebook(entries=entries, unit_width=unit), rb


def encode(codes, cb: Codebook) -> np.ndarray:
    """Gather one packed unit per code; absent symbols are corruption (huffman.py:193-203)."""
    codes = np.asarray(codes).reshape(-1)
    if codes.size == 0:
        return np.empty(0, dtype=cb.entries.dtype)
    _check_codes(codes, cb.cap)
    torch = _device._torch()
    d = _device.upload(codes.astype(np.uint32, copy=False).view(np.int32))
    ent = _device.upload(cb.entries.astype(np.uint64).view(np.int64))
    units = _device.empty(codes.size, torch.int32 if cb.unit_width == 32 else torch.int64)
    _lib.context().call("sdqz_encode_u32", _lib.ptr(d), codes.size, _lib.ptr(ent), cb.cap,
                        cb.unit_width, _lib.ptr(units))
    out = _device.download(units, codes.size)
    return out.view(np.uint32) if cb.unit_width == 32 else out.view(np.uint64)


def default_chunk_size(n_codes: int) -> int:
    """Codes per chunk aiming at ~2e4 chunks, clamped to [256, 65536] (huffman.py:206-212)."""
    if n_codes <= 0:
        return 256
    raw = n_codes / 2e4
    size = 1 << max(0, math.ceil(math.log2(raw))) if raw > 1 else 1
    return min(65536, max(256, size))


def deflate(packed, chunk_size: int) -> DeflatedStream:
    """Concatenate packed codewords MSB-first into byte-aligned chunks (huffman.py:219-269)."""
    if chunk_size < 1:
        raise SdqzError("chunk_size must be >= 1")
    packed = np.asarray(packed).reshape(-1)
    n = int(packed.size)
    if n == 0:
        return DeflatedStream(int(chunk_size), np.zeros(0, dtype=np.uint32), b"")
    unit = packed.dtype.itemsize * 8
    if unit not in (32, 64):
        packed = packed.astype(np.uint64)
        unit = 64
    torch = _device._torch()
    d = _device.upload(packed.view(np.int32 if unit == 32 else np.int64))
    nch = -(-n // chunk_size)
    bits = _device.empty(nch, torch.int32)
    cap_bytes = n * (unit // 8) + nch + 64
    pay = _device.empty(cap_bytes, torch.uint8)
    pb = _lib.c_uint64()
    _lib.context().call("sdqz_deflate_units", _lib.ptr(d), unit, n, int(chunk_size), _lib.ptr(bits),
                        _lib.ptr(pay), cap_bytes, _lib.byref(pb))
    return DeflatedStream(int(chunk_size), _device.download(bits, nch).view(np.uint32).copy(),
                          _device.download(pay, pb.value).tobytes())


def inflate(ds: DeflatedStream, rb: ReverseCodebook, n_codes: int,
            workers: int | None = None) -> np.ndarray:
    """Exact inverse of encode + deflate (huffman.py:311-356)."""
    bits = np.asarray(ds.chunk_bit_lengths, dtype=np.int64)
    n_chunks = int(bits.size)
    if n_codes == 0:
        if n_chunks or ds.payload:
            raise CorruptionError("nonempty stream for zero codes")
        return np.empty(0, dtype=CODE_DTYPE)
    if ds.chunk_size < 1 or n_chunks != -(-n_codes // ds.chunk_size):
        raise CorruptionError(f"{n_chunks} chunks inconsistent with {n_codes} codes of chunk "
                              f"size {ds.chunk_size}")
    need = int(((bits + 7) >> 3).sum())
    if need != len(ds.payload):
        raise CorruptionError(f"payload is {len(ds.payload)} bytes, chunk lengths require {need}")
    torch = _device._torch()
    pay = np.zeros(len(ds.payload) + 64, dtype=np.uint8)
    pay[: len(ds.payload)] = np.frombuffer(ds.payload, dtype=np.uint8)
    dpay = _device.upload(pay)
    dbits = _device.upload(bits.astype(np.uint32).view(np.int32))
    first = np.zeros(64, np.uint64)
    first[: rb.first_codes.size] = rb.first_codes
    offs = np.zeros(64, np.int64)
    offs[: rb.offsets.size] = rb.offsets
    offs[rb.offsets.size:] = rb.offsets[-1] if rb.offsets.size else 0
    syms = np.asarray(rb.symbols, dtype=np.uint32)
    dsym = _device.upload(np.concatenate([syms, np.zeros(1, np.uint32)]).view(np.int32))
    out = _device.empty(n_codes, torch.int32)
    dfirst = _device.upload(first.view(np.int64))   # keep references alive across the call
    doffs = _device.upload(offs)
    _lib.context().call("sdqz_inflate", _lib.ptr(dpay), len(ds.payload), _lib.ptr(dbits), n_chunks,
                        int(ds.chunk_size), _lib.ptr(dfirst), _lib.ptr(doffs), _lib.ptr(dsym),
                        int(rb.max_bitwidth), int(n_codes), _lib.ptr(out))
    return _device.download(out, n_codes).view(np.uint32).astype(CODE_DTYPE)
