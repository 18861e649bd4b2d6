# sdqz/_gpu.py -- the binding a maintainer of the reference package would add
# (INTEGRATION.md §2 shows this file verbatim; tests/test_integration_stub.py
# runs it).  It binds libsdqz_cuda.so's host-buffer entry points with ctypes:
# numpy in, bytes out, bytes in, numpy out -- no device allocator needed.
# Replaces the bodies of compress (sdqz/pipeline.py:15-39) and decompress
# (sdqz/pipeline.py:56-58).
import ctypes
import os

import numpy as np

try:                                            # inside the reference package
    from .archive import ArchiveFormatError
    from .core import CorruptionError, SdqzError
except ImportError:                             # standalone (the repo's tests)
    from paper_2007_09625_b200 import ArchiveFormatError, CorruptionError, SdqzError

_U64x3, _U32x3 = ctypes.c_uint64 * 3, ctypes.c_uint32 * 3


class _Hdr(ctypes.Structure):                  # sdqz_header (include/sdqz_cuda.h)
    _fields_ = [("dtype_code", ctypes.c_uint8), ("ndims", ctypes.c_uint8),
                ("eb_mode", ctypes.c_uint8), ("unit_width", ctypes.c_uint8),
                ("dims", _U64x3), ("eb_resolved", ctypes.c_double),
                ("eb_specified", ctypes.c_double), ("cap", ctypes.c_uint32),
                ("block", _U32x3), ("chunk_size", ctypes.c_uint32),
                ("n_outliers", ctypes.c_uint64), ("n_chunks", ctypes.c_uint64),
                ("payload_bytes", ctypes.c_uint64)]


_L = ctypes.CDLL(os.environ.get("SDQZ_CUDA_LIB", "libsdqz_cuda.so"))
_P, _I = ctypes.c_void_p, ctypes.c_int
_L.sdqz_ctx_create.argtypes = [_I, _P, ctypes.POINTER(_P)]
_L.sdqz_last_error.argtypes, _L.sdqz_last_error.restype = [_P], ctypes.c_char_p
_L.sdqz_archive_size.argtypes, _L.sdqz_archive_size.restype = [_P], ctypes.c_uint64   # > 2 GB archives
_L.sdqz_archive_write.argtypes = [_P, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_uint64]
_L.sdqz_compress_host.argtypes = [_P, _P, _I, _I, _U64x3, _U32x3, _I, ctypes.c_double, ctypes.c_uint32,
                                  ctypes.c_uint32, ctypes.POINTER(_Hdr)]
_L.sdqz_parse_header.argtypes = [_P, ctypes.c_char_p, ctypes.c_uint64, ctypes.POINTER(_Hdr)]
_L.sdqz_decompress_host.argtypes = [_P, ctypes.c_char_p, ctypes.c_uint64, _P]
for _f in ("sdqz_ctx_create", "sdqz_archive_write", "sdqz_compress_host", "sdqz_parse_header",
           "sdqz_decompress_host"):
    getattr(_L, _f).restype = _I
_ERR = {1: SdqzError, 2: CorruptionError, 3: ArchiveFormatError}
_ctx = _P()
if _L.sdqz_ctx_create(0, None, ctypes.byref(_ctx)):
    raise SdqzError("no CUDA device for libsdqz_cuda.so")


def _check(rc):
    if rc:
        raise _ERR.get(rc, SdqzError)(_L.sdqz_last_error(_ctx).decode())


def compress(data, dims=None, *, eb, mode="abs", cap=1024, block_shape=None, chunk_size=None,
             workers=None) -> bytes:
    if mode not in ("abs", "valrel"):                          # core.py:74-75
        raise SdqzError(f"unknown error-bound mode {mode!r} (use 'abs' or 'valrel')")
    a = np.ascontiguousarray(data)
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    dims = tuple(int(d) for d in (dims or (a.shape if a.ndim > 1 else (a.size,))))
    block = tuple(block_shape or {1: (32,), 2: (16, 16), 3: (8, 8, 8)}.get(len(dims), (1,)))
    h = _Hdr()
    _check(_L.sdqz_compress_host(_ctx, a.ctypes.data, int(a.dtype == np.float64), len(dims),
                                 _U64x3(*dims, *[1] * (3 - len(dims))),
                                 _U32x3(*block, *[1] * (3 - len(block))), int(mode == "valrel"),
                                 float(eb), int(cap), int(chunk_size or 0), ctypes.byref(h)))
    out = ctypes.create_string_buffer(_L.sdqz_archive_size(_ctx))
    _check(_L.sdqz_archive_write(_ctx, 0, out, len(out)))
    return out.raw


def decompress(blob: bytes, workers=None) -> np.ndarray:
    h = _Hdr()
    _check(_L.sdqz_parse_header(_ctx, blob, len(blob), ctypes.byref(h)))
    dims = tuple(h.dims[:h.ndims])
    out = np.empty(dims, np.float32 if h.dtype_code == 0 else np.float64)
    _check(_L.sdqz_decompress_host(_ctx, blob, len(blob), out.ctypes.data))
    return out
