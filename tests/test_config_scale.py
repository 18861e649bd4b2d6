"""Config-scale parity: BASELINE.json's configs at FULL size, bit-exact against
archives the REFERENCE itself produced (tests/golden/config_golden.json, made
by tests/golden/make_config_golden.py in the build container).

For every config the box first regenerates the reference's synthetic field and
proves it is the same field (SHA-256 of the fp32 input), then compresses on the
GPU and asserts the header fields, every archive section's SHA-256, the whole
archive's SHA-256, and the SHA-256 of the decompressed fp32 field.

  * CESM 1800x3600, Hurricane 100x500x500, HACC 280,953,867 (1D) and the Nyx
    512^3 sweep (valrel 1e-2..1e-5 x smooth / sparse-near-zero; smooth at 1e-3
    and 1e-4 has 27/25-bit codes -> 64-bit units) against the reference's
    whole-field compress / decompress;
  * 2048x2048x1024 (17.2 GB) against the reference's own row-slab
    decomposition of the same field (the workers>1 code path of compress_field /
    reconstruct_field, validated against the whole-field run on Nyx), hashed as
    digests of per-16-row-slab SHA-256s.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2007_09625_b200 as S  # noqa: E402
from paper_2007_09625_b200 import synthetic  # noqa: E402

CG = json.loads((Path(__file__).parent / "golden" / "config_golden.json").read_text())
WHOLE = sorted(k for k, v in CG.items() if "input_sha256" in v)


def sha(b) -> str:
    return hashlib.sha256(b).hexdigest()


def slab_digest(hashes) -> str:
    return sha("".join(hashes).encode())


def check_archive(blob: bytes, g: dict):
    h = S.parse_header(blob)
    got = {"cap": h.cap, "chunk_size": h.chunk_size, "unit_width": h.unit_width,
           "n_outliers": h.n_outliers, "n_chunks": h.n_chunks, "payload_bytes": h.payload_bytes,
           "archive_bytes": len(blob)}
    want = {k: g[k] for k in got}
    assert got == want
    assert np.float64(h.eb_resolved).tobytes().hex() == g["eb_resolved_hex"]
    p = S.HEADER_SIZE
    assert sha(blob[:p]) == g["sections"]["header"]
    for name, size in (("bitwidths", h.cap), ("outliers", 16 * h.n_outliers),
                       ("chunk_bits", 4 * h.n_chunks), ("payload", h.payload_bytes)):
        assert sha(blob[p:p + size]) == g["sections"][name], name
        p += size
    assert sha(blob) == g["archive_sha256"]


@pytest.mark.parametrize("name", WHOLE)
def test_config_matches_reference(name):
    g = CG[name]
    f = S.generate_field(g["profile"], tuple(g["dims"]), seed=g["seed"]).astype(np.float32)
    assert sha(f.tobytes()) == g["input_sha256"], "the box did not regenerate the reference's field"
    t = torch.from_numpy(f).cuda()
    del f
    dev = S.compress_device(t, eb=g["eb"], mode=g["mode"])
    check_archive(dev.to_bytes(), g)
    out = S.decompress_device(dev)
    assert sha(out.cpu().numpy().tobytes()) == g["output_sha256"]
    # and through the host-bytes API (archive bytes -> device decode)
    out2 = S.decompress_device(dev.to_bytes())
    assert torch.equal(out2.view(-1).view(torch.int32), out.view(-1).view(torch.int32))


def large_field_host(dims, rows=16):
    """The 2048x2048x1024 smooth field in pinned memory, bit-identical to the
    reference's generate_field (slab-wise on all cores), plus its per-slab digests."""
    n = math.prod(dims)
    inner = math.prod(dims[1:])
    pinned = torch.empty(n, dtype=torch.float32, pin_memory=True)
    arr = pinned.numpy()

    def fill(r0):
        a = synthetic.smooth_rows(dims, 1, (r0, r0 + rows)).astype(np.float32).reshape(-1)
        arr[r0 * inner:(r0 + rows) * inner] = a
        return sha(a.tobytes())

    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
        hashes = list(ex.map(fill, range(0, dims[0], rows)))
    return pinned, hashes


@pytest.mark.skipif("large" not in CG, reason="large golden not generated")
def test_large_matches_reference():
    g = CG["large"]
    dims, rows = tuple(g["dims"]), g["slab_rows"]
    inner = math.prod(dims[1:])
    pinned, hashes = large_field_host(dims, rows)
    assert slab_digest(hashes) == g["input_slab_digest"]
    t = pinned.cuda()
    del pinned
    dev = S.compress_device(t, dims, eb=g["eb"], mode=g["mode"])
    check_archive(dev.to_bytes(), g)
    del t
    out = S.decompress_device(dev).view(-1)
    host = torch.empty(rows * inner, dtype=torch.float32, pin_memory=True)
    outs = []
    for r0 in range(0, dims[0], rows):
        host.copy_(out[r0 * inner:(r0 + rows) * inner])
        outs.append(sha(host.numpy().tobytes()))
    assert slab_digest(outs) == g["output_slab_digest"]


def _large_sharded_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2007_09625_b200 import sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = CG["large"]
        dims = tuple(g["dims"])
        inner = math.prod(dims[1:])
        rows = sharded.slab_rows(dims[0], 8, world)
        r0 = sum(rows[:rank])
        slab = torch.empty(rows[rank] * inner, dtype=torch.float32, pin_memory=True)
        arr = slab.numpy()
        step = 16

        def fill(a):
            arr[a * inner:(a + step) * inner] = synthetic.smooth_rows(dims, 1, (r0 + a, r0 + a + step)) \
                .astype(np.float32).reshape(-1)

        with ThreadPoolExecutor(max_workers=max(1, 16 // world)) as ex:
            list(ex.map(fill, range(0, rows[rank], step)))
        d = slab.cuda().view((rows[rank],) + dims[1:])
        del slab, arr
        ar = sharded.compress_sharded_device(d, dims, eb=g["eb"], mode=g["mode"])
        blob = ar.gather(root=0)
        sha_ar = hashlib.sha256(blob).hexdigest() if blob is not None else None
        del blob
        # in-place decompress of this rank's slab: per-16-row-slab output digests
        out = sharded.decompress_sharded(ar, device=True).reshape(-1)
        host = torch.empty(16 * inner, dtype=torch.float32, pin_memory=True)
        hs = []
        for a in range(0, rows[rank], 16):
            host.copy_(out[a * inner:(a + 16) * inner])
            hs.append(sha(host.numpy().tobytes()))
        q.put((rank, sha_ar, hs, None))
    except Exception as e:  # surfaced by the parent
        q.put((rank, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif("large" not in CG, reason="large golden not generated")
@pytest.mark.parametrize("world", [2, 4])
def test_large_sharded_matches_reference(world):
    """The 17.2 GB field split over `world` ranks (gloo, sharing cuda:0): the
    assembled sharded archive and the in-place slab decompress equal the
    reference's archive and output (the same hashes as the single-GPU test)."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_large_sharded_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, sha_ar, hs, err = q.get(timeout=1200)
        res[r] = (sha_ar, hs, err)
    for p in procs:
        p.join(120)
    for r in range(world):
        assert res[r][2] is None, res[r][2]
    g = CG["large"]
    assert res[0][0] == g["archive_sha256"]
    assert slab_digest([h for r in range(world) for h in res[r][1]]) == g["output_slab_digest"]
