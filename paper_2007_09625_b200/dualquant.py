"""Lossy stage: dual-quantization around a blockwise Lorenzo predictor.

API mirror of the reference's dualquant module (sdqz/dualquant.py) -- names,
return types and error messages are the reference's -- with the work done by
the sm_100a kernels in csrc/dualquant.cu (prequant + Lorenzo + codes),
csrc/huffman.cu (ordered outlier compaction) and csrc/reconstruct.cu
(exact integer Lorenzo inverse).  `pad_block` / `lorenzo_predict` are the
reference's single-block/single-point helpers and stay scalar host code; the
block-level `postquantize_block` runs the same device kernel as whole fields.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from .core import CorruptionError, FieldDescriptor, QuantConfig, SdqzError, partition_blocks

CODE_DTYPE = np.uint32


@dataclass
class PrequantField:
    """Values snapped to the 2*eb lattice, exact integers in float64 (dualquant.py:31-39)."""

    values: np.ndarray
    dims: tuple[int, ...]

    @property
    def shaped(self) -> np.ndarray:
        return self.values.reshape(self.dims)


@dataclass
class QuantOutput:
    """Codes (0 = outlier) plus the verbatim outlier list (dualquant.py:42-59)."""

    codes: np.ndarray            # uint32, flat
    outlier_indices: np.ndarray  # uint64, strictly ascending flat indices
    outlier_values: np.ndarray   # float64, prequantized units
    dims: tuple[int, ...]
    cfg: QuantConfig

    @property
    def n_outliers(self) -> int:
        return int(self.outlier_indices.size)


def prequantize(data, eb: float, dims: tuple[int, ...] | None = None) -> PrequantField:
    """x / (2 eb) rounded half away from zero, fp64 (dualquant.py:62-78)."""
    arr = _device.as_field(data)
    if not (eb > 0 and math.isfinite(eb)):
        raise SdqzError("error bound must be positive")
    if dims is None:
        shape = tuple(arr.shape)
        dims = shape if len(shape) > 1 else (_device.numel(arr),)
    t, dt = _device.to_device(arr)
    n = t.numel()
    if n:
        _, _, nonfinite = _device.describe(t, dt)
        if nonfinite:
            raise SdqzError("cannot prequantize nonfinite values")
    torch = _device._torch()
    out = _device.empty(n, torch.float64)
    if n:
        _lib.context().call("sdqz_prequantize", _lib.ptr(t), 0 if dt == np.float32 else 1, n,
                            float(eb), _lib.ptr(out))
    return PrequantField(values=_device.download(out, n), dims=tuple(int(d) for d in dims))


def pad_block(block: np.ndarray) -> np.ndarray:
    """One block's prediction context: a leading zero layer per axis (dualquant.py:81-86)."""
    block = np.asarray(block, dtype=np.float64)
    out = np.zeros(tuple(e + 1 for e in block.shape))
    out[(slice(1, None),) * block.ndim] = block
    return out


def lorenzo_predict(padded: np.ndarray, coords: tuple[int, ...]) -> float:
    """First-order Lorenzo prediction of one point (dualquant.py:89-112)."""
    r = padded.ndim
    if len(coords) != r:
        raise SdqzError(f"got {len(coords)} coordinates for a rank-{r} context")
    p = padded
    if r == 1:
        (a,) = coords
        return float(p[a])
    if r == 2:
        a, b = coords
        return float(p[a, b + 1] + p[a + 1, b] - p[a, b])
    if r == 3:
        a, b, c = coords
        return float(p[a, b + 1, c + 1] + p[a + 1, b, c + 1] + p[a + 1, b + 1, c]
                     - p[a, b, c + 1] - p[a, b + 1, c] - p[a + 1, b, c] + p[a, b, c])
    raise SdqzError(f"rank {r} not supported (1-3)")


def _codes_device(t, in_kind: int, dims, cfg: QuantConfig, want_hist: bool):
    torch = _device._torch()
    n = math.prod(dims)
    codes = _device.empty(n + 8, torch.int16)
    hist = _device.empty(cfg.cap, torch.int64) if want_hist else None
    nf = _lib.c_int()
    _lib.context().call("sdqz_dualquant", _lib.ptr(t), in_kind, len(dims), _lib.dims3(dims),
                        _lib.block3(cfg.block_shape), float(cfg.eb), int(cfg.cap),
                        _lib.ptr(codes), _lib.ptr(hist), _lib.byref(nf))
    return codes, hist, bool(nf.value)


def _outliers_device(t, in_kind: int, codes, n: int, eb: float):
    torch = _device._torch()
    rec = _device.empty(2 * n + 2, torch.int64)
    k = _lib.c_uint64()
    _lib.context().call("sdqz_outliers", _lib.ptr(t), in_kind, _lib.ptr(codes), n, float(eb),
                        _lib.ptr(rec), n + 1, _lib.byref(k))
    r = _device.download(rec[: 2 * k.value]).view(np.uint64).reshape(-1, 2)
    return r[:, 0].copy(), r[:, 1].copy().view(np.float64)


def _codes_u32(codes_dev, n):
    return (_device.download(codes_dev, n).view(np.uint16)).astype(CODE_DTYPE)


def postquantize_block(padded: np.ndarray, cfg: QuantConfig):
    """Residual-code one padded block of prequantized values (dualquant.py:132-147).

    Returns (codes shaped like the block, local outlier indices, values)."""
    padded = np.asarray(padded, dtype=np.float64)
    inner = np.ascontiguousarray(padded[(slice(1, None),) * padded.ndim])
    dims = inner.shape
    local_cfg = QuantConfig(eb=cfg.eb, cap=cfg.cap, block_shape=dims)
    t = _device.upload(inner)
    codes, _, _ = _codes_device(t, 2, dims, local_cfg, False)
    n = inner.size
    c = _codes_u32(codes, n)
    idx = np.flatnonzero(c == 0)
    return c.reshape(dims), idx, inner.reshape(-1)[idx]


def compress_field(data, fd: FieldDescriptor, cfg: QuantConfig,
                   workers: int | None = None) -> QuantOutput:
    """Prequantize + residual-code a whole field (dualquant.py:242-273).

    `workers` is accepted for API compatibility; the output never depends on
    it (dualquant.py:245-248)."""
    partition_blocks(fd, cfg)
    arr = _device.as_field(data)
    if _device.numel(arr) != fd.n_points:
        raise SdqzError(f"data has {_device.numel(arr)} values, descriptor expects {fd.n_points}")
    t, dt = _device.to_device(arr)
    kind = 0 if dt == np.float32 else 1
    codes, _, nonfinite = _codes_device(t, kind, fd.dims, cfg, False)
    if nonfinite:
        raise SdqzError("cannot prequantize nonfinite values")
    idx, vals = _outliers_device(t, kind, codes, fd.n_points, cfg.eb)
    return QuantOutput(_codes_u32(codes, fd.n_points), idx.astype(np.uint64),
                       vals.astype(np.float64), fd.dims, cfg)


def reconstruct_field(qout: QuantOutput, cfg: QuantConfig | None = None,
                      workers: int | None = None) -> np.ndarray:
    """Rebuild the field from codes + outliers: flat float64, |err| <= eb
    (dualquant.py:299-332), validated like _validate_output (:276-296)."""
    cfg = cfg or qout.cfg
    n = math.prod(qout.dims)
    codes = np.asarray(qout.codes)
    if codes.size != n:
        raise CorruptionError(f"code array has {codes.size} entries, expected {n}")
    idx = np.asarray(qout.outlier_indices)
    vals = np.asarray(qout.outlier_values, dtype=np.float64)
    if idx.size != vals.size:
        raise CorruptionError("outlier index/value lengths differ")
    torch = _device._torch()
    if codes.dtype.itemsize > 4 or (codes.size and codes.dtype.kind == "i" and int(codes.min()) < 0):
        if codes.size and (int(codes.min()) < 0 or int(codes.max()) >= cfg.cap):
            raise CorruptionError("quantization code out of range for cap")
    c32 = _device.upload(codes.astype(np.uint32, copy=False).view(np.int32))
    di = _device.upload(idx.astype(np.uint64).view(np.int64)) if idx.size else None
    dv = _device.upload(vals) if idx.size else None
    out = _device.empty(n, torch.float64)
    _lib.context().call("sdqz_reconstruct", _lib.ptr(c32), 4, n, _lib.ptr(di), _lib.ptr(dv),
                        int(idx.size), len(qout.dims), _lib.dims3(qout.dims),
                        _lib.block3(cfg.block_shape), float(cfg.eb), int(cfg.cap), _lib.ptr(out), 1)
    return _device.download(out, n)
