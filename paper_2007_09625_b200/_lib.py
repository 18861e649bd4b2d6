"""ctypes binding of libsdqz_cuda.so (include/sdqz_cuda.h).

There is no CPU fallback: if the shared library is missing the import of the
package's compute entry points fails loudly, and every compute call needs a
CUDA device.  Device buffers are torch tensors (torch is only the allocator /
stream plumbing); the library sees plain pointers.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import (POINTER, Structure, byref, c_char_p, c_double, c_int, c_int64, c_uint8,
                    c_uint32, c_uint64, c_void_p)
from pathlib import Path

from .core import CorruptionError, SdqzError

# SDQZ_LIB_PATH: load another build of the same library (A/B kernel experiments)
LIB_PATH = Path(os.environ.get("SDQZ_LIB_PATH") or Path(__file__).resolve().parent / "libsdqz_cuda.so")

SDQZ_OK, SDQZ_EINVAL, SDQZ_ECORRUPT, SDQZ_EFORMAT, SDQZ_ECUDA = range(5)
HEADER_SIZE = 93


class Header(Structure):
    """sdqz_header (include/sdqz_cuda.h)."""

    _fields_ = [
        ("dtype_code", c_uint8), ("ndims", c_uint8), ("eb_mode", c_uint8), ("unit_width", c_uint8),
        ("dims", c_uint64 * 3), ("eb_resolved", c_double), ("eb_specified", c_double),
        ("cap", c_uint32), ("block", c_uint32 * 3), ("chunk_size", c_uint32),
        ("n_outliers", c_uint64), ("n_chunks", c_uint64), ("payload_bytes", c_uint64),
    ]

    def copy(self) -> "Header":
        h = Header()
        ctypes.pointer(h)[0] = self
        return h

    @property
    def total_bytes(self) -> int:
        return (HEADER_SIZE + self.cap + 16 * self.n_outliers + 4 * self.n_chunks
                + self.payload_bytes)


class ShardSizes(Structure):
    """sdqz_shard_sizes (include/sdqz_cuda.h)."""

    _fields_ = [("n_chunks", c_uint64), ("payload_bytes", c_uint64), ("n_outliers", c_uint64),
                ("unit_width", c_uint32), ("max_bw", c_uint32), ("eb_resolved", c_double)]


_SIGS = {
    "sdqz_ctx_create": (c_int, [c_int, c_void_p, POINTER(c_void_p)]),
    "sdqz_ctx_destroy": (c_int, [c_void_p]),
    "sdqz_ctx_set_stream": (c_int, [c_void_p, c_void_p]),
    "sdqz_last_error": (c_char_p, [c_void_p]),
    "sdqz_kernel_launches": (c_uint64, [c_void_p]),
    "sdqz_graph_replays": (c_uint64, [c_void_p]),
    "sdqz_set_timing": (c_int, [c_void_p, c_int]),
    "sdqz_debug_counters": (c_int, [c_void_p, POINTER(c_uint64), c_int]),
    "sdqz_debug_read": (c_int, [c_void_p, c_int, c_void_p, c_uint64]),
    "sdqz_kernel_times": (c_int, [c_void_p, c_char_p, c_uint64]),
    "sdqz_describe": (c_int, [c_void_p, c_void_p, c_int, c_uint64, POINTER(c_double),
                              POINTER(c_double), POINTER(c_int)]),
    "sdqz_prequantize": (c_int, [c_void_p, c_void_p, c_int, c_uint64, c_double, c_void_p]),
    "sdqz_upload": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p]),
    "sdqz_quality": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_int, c_uint64, POINTER(c_double)]),
    "sdqz_dualquant": (c_int, [c_void_p, c_void_p, c_int, c_int, POINTER(c_uint64),
                               POINTER(c_uint32), c_double, c_uint32, c_void_p, c_void_p,
                               POINTER(c_int)]),
    "sdqz_outliers": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_uint64, c_double, c_void_p,
                              c_uint64, POINTER(c_uint64)]),
    "sdqz_reconstruct": (c_int, [c_void_p, c_void_p, c_int, c_uint64, c_void_p, c_void_p,
                                 c_uint64, c_int, POINTER(c_uint64), POINTER(c_uint32), c_double,
                                 c_uint32, c_void_p, c_int]),
    "sdqz_histogram_u32": (c_int, [c_void_p, c_void_p, c_uint64, c_uint32, c_void_p]),
    "sdqz_build_tree": (c_int, [c_void_p, c_void_p, c_uint32, c_void_p]),
    "sdqz_canonize": (c_int, [c_void_p, c_void_p, c_uint32, c_void_p, c_void_p, c_void_p,
                              c_void_p, POINTER(c_int), POINTER(c_int), POINTER(c_uint32)]),
    "sdqz_encode_u32": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p, c_uint32, c_int,
                                c_void_p]),
    "sdqz_deflate_units": (c_int, [c_void_p, c_void_p, c_int, c_uint64, c_uint32, c_void_p,
                                   c_void_p, c_uint64, POINTER(c_uint64)]),
    "sdqz_encode_deflate": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p, c_uint32, c_uint32,
                                    c_void_p, c_void_p, c_uint64, POINTER(c_uint64)]),
    "sdqz_inflate": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p, c_uint64, c_uint32,
                             c_void_p, c_void_p, c_void_p, c_int, c_uint64, c_void_p]),
    "sdqz_compress": (c_int, [c_void_p, c_void_p, c_int, c_int, POINTER(c_uint64),
                              POINTER(c_uint32), c_int, c_double, c_uint32, c_uint32,
                              POINTER(Header)]),
    "sdqz_compress_described": (c_int, [c_void_p, c_void_p, c_int, c_int, POINTER(c_uint64),
                                        POINTER(c_uint32), c_int, c_double, c_uint32, c_uint32,
                                        POINTER(c_double), POINTER(Header)]),
    "sdqz_archive_size": (c_uint64, [c_void_p]),
    "sdqz_archive_generation": (c_uint64, [c_void_p]),
    "sdqz_archive_write": (c_int, [c_void_p, c_uint64, c_void_p, c_uint64]),
    "sdqz_archive_copy": (c_int, [c_void_p, c_uint64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sdqz_archive_sections": (c_int, [c_void_p, c_uint64, POINTER(c_void_p), POINTER(c_void_p),
                                      POINTER(c_void_p), POINTER(c_void_p)]),
    "sdqz_parse_header": (c_int, [c_void_p, c_void_p, c_uint64, POINTER(Header)]),
    "sdqz_decompress": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p]),
    "sdqz_decompress_sections": (c_int, [c_void_p, POINTER(Header), c_void_p, c_void_p,
                                         c_void_p, c_void_p, c_void_p]),
    "sdqz_decompress_slab": (c_int, [c_void_p, POINTER(Header), c_void_p, c_void_p, c_uint64, c_uint64,
                                     c_void_p, c_uint64, c_void_p, c_uint64, c_uint64, c_uint64,
                                     POINTER(c_uint64), c_void_p]),
    "sdqz_decompress_quality": (c_int, [c_void_p, POINTER(Header), c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_void_p, c_int, POINTER(c_double), POINTER(c_int)]),
    "sdqz_device_count": (c_int, [POINTER(c_int)]),
    "sdqz_compress_host": (c_int, [c_void_p, c_void_p, c_int, c_int, POINTER(c_uint64),
                                   POINTER(c_uint32), c_int, c_double, c_uint32, c_uint32,
                                   POINTER(Header)]),
    "sdqz_decompress_host": (c_int, [c_void_p, c_void_p, c_uint64, c_void_p]),
    "sdqz_quality_host": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_int, c_uint64,
                                  POINTER(c_double)]),
    "sdqz_shard_describe": (c_int, [c_void_p, c_void_p, c_int, c_uint64, c_void_p]),
    "sdqz_shard_quantize": (c_int, [c_void_p, c_void_p, c_int, c_int, POINTER(c_uint64), POINTER(c_uint32),
                                    c_int, c_double, c_uint32, c_void_p, c_void_p]),
    "sdqz_shard_head": (c_int, [c_void_p, c_uint64, c_void_p]),
    "sdqz_shard_encode": (c_int, [c_void_p, c_void_p, c_uint32, c_uint64, c_void_p, c_uint64, c_uint64,
                                  POINTER(ShardSizes)]),
}

EXPORTS = tuple(_SIGS)

_lib = None
_lib_lock = threading.Lock()


def load_library():
    """Load libsdqz_cuda.so (no GPU needed for loading).  Raises if absent."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (or make -C paper_2007_09625_b200/csrc). There is no CPU "
                    f"fallback for the sdqz compute path.")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def _exc_for(rc: int, msg: str):
    from .archive import ArchiveFormatError
    if rc == SDQZ_ECORRUPT:
        return CorruptionError(msg)
    if rc == SDQZ_EFORMAT:
        return ArchiveFormatError(msg)
    if rc == SDQZ_EINVAL:
        return SdqzError(msg)
    return RuntimeError(f"sdqz CUDA failure: {msg}")


class Context:
    """One library context per (device, host thread): stream + scratch arena."""

    def __init__(self, device: int):
        import torch
        self.lib = load_library()
        self.device = device
        self.torch = torch
        h = c_void_p()
        rc = self.lib.sdqz_ctx_create(device, c_void_p(torch.cuda.current_stream(device).cuda_stream),
                                      byref(h))
        if rc:
            raise RuntimeError(f"sdqz_ctx_create failed ({rc}) on cuda:{device}")
        self.h = h

    def sync_stream(self):
        s = self.torch.cuda.current_stream(self.device).cuda_stream
        self.lib.sdqz_ctx_set_stream(self.h, c_void_p(s))

    def call(self, name: str, *args):
        rc = getattr(self.lib, name)(self.h, *args)
        if rc != SDQZ_OK:
            msg = self.lib.sdqz_last_error(self.h).decode(errors="replace")
            raise _exc_for(rc, msg)
        return rc

    def set_timing(self, on: bool) -> None:
        self.lib.sdqz_set_timing(self.h, 1 if on else 0)

    def kernel_times(self) -> dict:
        """Accumulated device ms per kernel name since set_timing(True)."""
        buf = ctypes.create_string_buffer(8192)
        self.lib.sdqz_kernel_times(self.h, buf, 8192)
        out = {}
        for item in buf.value.decode().split(";"):
            if "=" in item:
                k, v = item.split("=")
                out[k] = float(v)
        return out

    @property
    def archive_generation(self) -> int:
        return int(self.lib.sdqz_archive_generation(self.h))

    @property
    def launches(self) -> int:
        return int(self.lib.sdqz_kernel_launches(self.h))

    @property
    def graph_replays(self) -> int:
        return int(self.lib.sdqz_graph_replays(self.h))

    def __del__(self):  # pragma: no cover - interpreter shutdown order varies
        try:
            if getattr(self, "h", None):
                self.lib.sdqz_ctx_destroy(self.h)
        except Exception:
            pass


class HostContext(Context):
    """A context with its own CUDA stream and no torch: for the host-buffer
    entry points (sdqz_*_host), e.g. the CLI, which then never imports torch."""

    def __init__(self, device: int):  # noqa: D401 - no torch here
        self.lib = load_library()
        self.device = device
        self.torch = None
        h = c_void_p()
        rc = self.lib.sdqz_ctx_create(device, None, byref(h))
        if rc:
            raise RuntimeError(f"sdqz_ctx_create failed ({rc}) on cuda:{device}")
        self.h = h

    def sync_stream(self):
        pass


_tls = threading.local()


def host_context() -> HostContext:
    """The calling thread's torch-free context (device: torch's current one if
    torch is loaded, else $SDQZ_DEVICE or 0).  Raises without a CUDA device."""
    import sys
    lib = load_library()
    n = c_int(0)
    lib.sdqz_device_count(byref(n))
    if n.value < 1:
        raise RuntimeError("sdqz (B200 build) needs a CUDA device; no CPU fallback exists")
    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_initialized():
        device = torch.cuda.current_device()
    else:
        device = int(os.environ.get("SDQZ_DEVICE", "0"))
    hc = getattr(_tls, "hctx", None)
    if hc is None:
        hc = _tls.hctx = {}
    ctx = hc.get(device)
    if ctx is None:
        ctx = hc[device] = HostContext(device)
    return ctx


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("sdqz (B200 build) needs a CUDA device; no CPU fallback exists")
    load_library()


def context(device: int | None = None) -> Context:
    """The calling thread's context for `device` (default: torch's current device)."""
    import torch
    require_cuda()
    if device is None:
        device = torch.cuda.current_device()
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    ctx = ctxs.get(device)
    if ctx is None:
        with torch.cuda.device(device):
            ctx = ctxs[device] = Context(device)
    ctx.sync_stream()
    return ctx


def dims3(dims):
    d = list(int(x) for x in dims) + [1] * (3 - len(dims))
    return (c_uint64 * 3)(*d)


def block3(block):
    b = list(int(x) for x in block) + [1] * (3 - len(block))
    return (c_uint32 * 3)(*b)


def ptr(t) -> c_void_p:
    return c_void_p(t.data_ptr()) if t is not None else c_void_p(0)


def env_flag(name: str) -> bool:
    return os.environ.get(name, "") not in ("", "0")


__all__ = ["Context", "Header", "ShardSizes", "EXPORTS", "LIB_PATH", "load_library", "context", "dims3",
           "block3", "ptr", "require_cuda", "c_int", "c_uint32", "c_uint64", "c_double",
           "c_int64", "byref", "c_void_p"]
