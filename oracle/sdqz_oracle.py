"""CPU oracle for the sdqz compression path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_2007_09625_b200/`) imports, links or executes this module; only
`tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference`
legs of `bench.py` may use it, and there only as the checker (or as the timed
CPU baseline), never as the thing measured for the GPU arm.

This is a numpy restatement of the reference package `sdqz`
(/root/reference/pkg/src/sdqz, pure Python + numpy).  Every function cites the
reference file:line whose behaviour it restates.  It is pinned (see
tests/test_oracle.py) against:
  * the golden archive SHA-256 pinned by the reference's own acceptance test
    (tests/test_acceptance.py:26, recipe :221-227), and
  * stage-level and archive-level golden vectors produced by importing the
    reference itself in the build container (tests/golden/make_golden.py).

Arithmetic contract (identical to the reference):
  * prequant: IEEE fp64 *division* x/(2eb), floor(|x|+0.5), copysign
    (keeps -0.0 for outlier payloads);
  * Lorenzo predictor evaluated in fp64 in the reference's term order;
  * reconstruction: blockwise cumsum per axis (fp64) then one correction per
    outlier in raster order, x (2eb) in fp64, cast to the archive dtype.
"""

from __future__ import annotations

import heapq  # noqa: F401  (documented alternative; two-queue merge used below)
import math
import struct
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

# --------------------------------------------------------------------------
# errors / constants  (core.py:15-31, archive.py:31-45)
# --------------------------------------------------------------------------


class OracleError(Exception):
    """Mirror of sdqz.SdqzError (core.py:26)."""


class OracleCorruption(OracleError):
    """Mirror of sdqz.CorruptionError (core.py:30)."""


class OracleFormatError(OracleError):
    """Mirror of sdqz.ArchiveFormatError (archive.py:44)."""


DEFAULT_BLOCKS = {1: (32,), 2: (16, 16), 3: (8, 8, 8)}       # core.py:16-20
HEADER = struct.Struct("<4s4B3Q2d5IB3Q")                     # archive.py:34
HEADER_SIZE = HEADER.size                                    # 93
MAGIC = b"SDQZ"


# --------------------------------------------------------------------------
# L1: describe / error bound / chunk size
# --------------------------------------------------------------------------

def describe(data):
    """min, max (in the input's float dtype, returned as Python floats) and the
    nonfinite flag; non-float input is promoted to float64 (core.py:136-158)."""
    a = np.asarray(data)
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    flat = a.reshape(-1)
    if flat.size == 0:
        raise OracleError("empty field")
    return float(flat.min()), float(flat.max()), not bool(np.isfinite(flat).all()), a.dtype


def resolve_eb(mode, magnitude, vmin, vmax, nonfinite):
    """core.py:161-175 (checks in the same order, same wording)."""
    if nonfinite:
        raise OracleError("field contains NaN/Inf values and cannot be compressed")
    if not (magnitude > 0 and math.isfinite(magnitude)):
        raise OracleError("error bound must be positive")
    if mode == "abs":
        return float(magnitude)
    rng = vmax - vmin
    if rng == 0.0:
        raise OracleError("value-range-relative bound is undefined on a constant field; "
                          "use an absolute error bound instead")
    return float(magnitude) * rng


def default_chunk_size(n):
    """huffman.py:206-212: 2^ceil(log2(n/2e4)) clamped to [256, 65536]."""
    if n <= 0:
        return 256
    q = n / 2e4
    e = math.ceil(math.log2(q)) if q > 1 else 0
    return int(min(65536, max(256, 1 << max(0, e))))


# --------------------------------------------------------------------------
# L2 lossy: prequant + blockwise Lorenzo  (dualquant.py:62-194)
# --------------------------------------------------------------------------

def prequant(data, eb):
    """dualquant.py:76-77 -- fp64 division, half-away-from-zero rounding."""
    x = np.asarray(data).astype(np.float64).reshape(-1) / (2.0 * eb)
    return np.copysign(np.floor(np.abs(x) + 0.5), x)


def _shift(f, axis, block):
    """Neighbour at coordinate-1 along `axis`, zero where the point sits on a
    block's leading face (the zero pad of dualquant.py:81-86, :185-186)."""
    out = np.zeros_like(f)
    src = [slice(None)] * f.ndim
    dst = [slice(None)] * f.ndim
    src[axis] = slice(0, f.shape[axis] - 1)
    dst[axis] = slice(1, f.shape[axis])
    out[tuple(dst)] = f[tuple(src)]
    lead = (np.arange(f.shape[axis]) % block) == 0
    idx = [slice(None)] * f.ndim
    idx[axis] = lead
    out[tuple(idx)] = 0.0
    return out


def lorenzo_pred(dq, block):
    """Prediction of every point, fp64, terms in the reference's order
    (dualquant.py:115-129): 1D p=(a-1); 2D (a-1,b)+(a,b-1)-(a-1,b-1);
    3D +(a-1,b,c)+(a,b-1,c)+(a,b,c-1)-(a-1,b-1,c)-(a-1,b,c-1)-(a,b-1,c-1)+(a-1,b-1,c-1)."""
    r = dq.ndim
    if r == 1:
        return _shift(dq, 0, block[0])
    if r == 2:
        sa = _shift(dq, 0, block[0])
        sb = _shift(dq, 1, block[1])
        sab = _shift(sa, 1, block[1])
        return sa + sb - sab
    sa = _shift(dq, 0, block[0])
    sb = _shift(dq, 1, block[1])
    sc = _shift(dq, 2, block[2])
    sab = _shift(sa, 1, block[1])
    sac = _shift(sa, 2, block[2])
    sbc = _shift(sb, 2, block[2])
    sabc = _shift(sab, 2, block[2])
    return sa + sb + sc - sab - sac - sbc + sabc


def dualquant(data, dims, eb, cap, block):
    """compress_field (dualquant.py:242-273 / _compress_region :172-194).

    Returns codes (uint32, flat), outlier indices (uint64, ascending global
    row-major) and outlier values (fp64 prequant units, -0.0 preserved)."""
    dims = tuple(int(d) for d in dims)
    radius = cap // 2
    dq = prequant(data, eb).reshape(dims)
    delta = dq - lorenzo_pred(dq, block)
    keep = (delta > -radius) & (delta < radius)
    codes = np.where(keep, delta + radius, 0.0).astype(np.uint32).reshape(-1)
    idx = np.flatnonzero(~keep.reshape(-1))
    return codes, idx.astype(np.uint64), dq.reshape(-1)[idx].astype(np.float64)


def _block_view_cumsum(res, block):
    """Blockwise inclusive cumsum along every axis, axis 0 first
    (dualquant.py:215-217).  `res` is already padded to whole blocks."""
    r = res.ndim
    shape = []
    for d, b in zip(res.shape, block):
        shape += [d // b, b]
    v = res.reshape(shape)
    for ax in range(r):
        v = np.cumsum(v, axis=2 * ax + 1)
    return v.reshape(res.shape)


def reconstruct(codes, out_idx, out_val, dims, eb, cap, block):
    """reconstruct_field (dualquant.py:299-332 / _reconstruct_region :197-227):
    in-cap residuals -> blockwise cumsum; each outlier, in global raster
    order, adds (value - current) over the trailing box of its block; then
    x (2eb) in fp64.  Returns flat fp64."""
    dims = tuple(int(d) for d in dims)
    radius = cap // 2
    c = np.asarray(codes).reshape(dims)
    padded = tuple(-(-d // b) * b for d, b in zip(dims, block))
    res = np.zeros(padded)
    region = tuple(slice(0, d) for d in dims)
    res[region] = np.where(c == 0, 0.0, c.astype(np.float64) - radius)
    acc = _block_view_cumsum(res, block)
    idx = np.asarray(out_idx, dtype=np.int64)
    if idx.size:
        coords = np.unravel_index(idx, dims)
        vals = np.asarray(out_val, dtype=np.float64).tolist()
        cl = [cc.tolist() for cc in coords]
        for k, v in enumerate(vals):
            p = tuple(cl[a][k] for a in range(len(dims)))
            box = tuple(slice(p[a], (p[a] // block[a] + 1) * block[a]) for a in range(len(dims)))
            acc[box] += v - acc[p]
    return acc[region].reshape(-1) * (2.0 * eb)


def validate_quant(codes, out_idx, out_val, n, cap):
    """_validate_output (dualquant.py:276-296), same order and wording."""
    codes = np.asarray(codes)
    if codes.size != n:
        raise OracleCorruption(f"code array has {codes.size} entries, expected {n}")
    if codes.size and int(codes.max()) >= cap:
        raise OracleCorruption("quantization code out of range for cap")
    idx = np.asarray(out_idx)
    if idx.size != np.asarray(out_val).size:
        raise OracleCorruption("outlier index/value lengths differ")
    if idx.size:
        if int(idx.max()) >= n:
            raise OracleCorruption("outlier index out of range")
        if np.any(np.diff(idx.astype(np.int64)) <= 0):
            raise OracleCorruption("outlier indices must be strictly ascending")
        if np.any(codes[idx.astype(np.int64)] != 0):
            raise OracleCorruption("outlier entry at a position whose code is not 0")
    zeros = int(np.count_nonzero(codes == 0))
    if zeros != idx.size:
        raise OracleCorruption(f"{zeros} zero codes but {idx.size} outlier entries")


# --------------------------------------------------------------------------
# L2 lossless: histogram, tree, canonical codebook, deflate/inflate
# --------------------------------------------------------------------------

def histogram(codes, cap):
    """huffman.py:77-95 (exact int64 counts; code >= cap is corruption)."""
    c = np.asarray(codes).reshape(-1)
    if c.size == 0:
        return np.zeros(cap, dtype=np.int64)
    if int(c.min()) < 0 or int(c.max()) >= cap:
        raise OracleCorruption(f"quantization code outside [0, {cap})")
    return np.bincount(c, minlength=cap).astype(np.int64)


def tree_bitwidths(freq):
    """build_tree (huffman.py:98-131).  The reference pops a heap keyed by
    (weight, smallest contained symbol).  Restated as the classic two-queue
    merge over leaves sorted by (freq, symbol): with integer weights >= 1,
    internal nodes are created in strictly increasing (weight, minsym) order,
    so comparing queue heads on that key reproduces the heap's pop sequence
    exactly (pinned by the golden tree vectors)."""
    f = np.asarray(freq, dtype=np.int64)
    syms = np.flatnonzero(f > 0)
    out = np.zeros(f.size, dtype=np.uint8)
    if syms.size == 0:
        raise OracleError("cannot build a code from an all-zero histogram")
    if syms.size == 1:
        out[syms[0]] = 1
        return out
    order = np.lexsort((syms, f[syms]))
    leaves = syms[order]
    lw = f[leaves].tolist()
    ls = leaves.tolist()
    n = len(ls)
    parent = [0] * (2 * n - 1)
    iw, im = [], []          # internal queue: weight, minsym (node id = n + pos)
    li = ii = 0
    for k in range(n - 1):
        pick = []
        for _ in range(2):
            take_leaf = ii >= len(iw) or (li < n and (lw[li], ls[li]) < (iw[ii], im[ii]))
            if take_leaf:
                pick.append((lw[li], ls[li], li))
                li += 1
            else:
                pick.append((iw[ii], im[ii], n + ii))
                ii += 1
        (w1, m1, a), (w2, m2, b) = pick
        parent[a] = parent[b] = n + k
        iw.append(w1 + w2)
        im.append(min(m1, m2))
    depth = [0] * (2 * n - 1)
    for node in range(2 * n - 3, -1, -1):
        depth[node] = depth[parent[node]] + 1
    for j in range(n):
        out[ls[j]] = depth[j] & 0xFF
    return out


def unit_width(max_bw):
    """select_unit_width (huffman.py:134-143)."""
    if max_bw < 1:
        raise OracleError("maximum bitwidth must be >= 1")
    if max_bw > 56:
        raise OracleError(f"codeword bitwidth {max_bw} exceeds the supported maximum of 56")
    return 32 if max_bw <= 24 else 64


@dataclass
class Book:
    entries: np.ndarray      # u32 or u64 packed (bw << (unit-8)) | codeword
    unit: int
    first: np.ndarray        # u64 per width
    offsets: np.ndarray      # i64 per width (+1 sentinel)
    symbols: np.ndarray      # u32 sorted by (width, symbol)
    max_bw: int


def canonical_book(bitwidths):
    """canonize (huffman.py:146-190): Kraft check, lexsort((sym, bw)),
    first_codes recurrence, packed entries."""
    bw = np.asarray(bitwidths, dtype=np.uint8)
    syms = np.flatnonzero(bw)
    if syms.size == 0:
        raise OracleError("cannot canonize an empty codebook")
    w = bw[syms].astype(np.int64)
    mx = int(w.max())
    unit = unit_width(mx)
    cnt = np.bincount(w, minlength=mx + 1)
    if syms.size >= 2:
        total = 0
        for b in range(1, mx + 1):
            total += int(cnt[b]) << (mx - b)
        if total != (1 << mx):
            raise OracleError("bitwidth table violates Kraft equality")
    order = np.lexsort((syms, w))
    sorted_syms = syms[order]
    sorted_w = w[order]
    first = np.zeros(mx + 1, dtype=np.uint64)
    run = 0
    for b in range(2, mx + 1):
        run = (run + int(cnt[b - 1])) << 1
        first[b] = run
    offs = np.zeros(mx + 2, dtype=np.int64)
    offs[1:] = np.cumsum(cnt)
    rank = np.arange(sorted_syms.size, dtype=np.int64) - offs[sorted_w]
    cw = first[sorted_w] + rank.astype(np.uint64)
    packed = (sorted_w.astype(np.uint64) << np.uint64(unit - 8)) | cw
    entries = np.zeros(bw.size, dtype=np.uint64)
    entries[sorted_syms] = packed
    if unit == 32:
        entries = entries.astype(np.uint32)
    return Book(entries, unit, first, offs, sorted_syms.astype(np.uint32), mx)


def encode(codes, book):
    """huffman.py:193-203."""
    c = np.asarray(codes).reshape(-1)
    if c.size == 0:
        return np.empty(0, dtype=book.entries.dtype)
    if int(c.min()) < 0 or int(c.max()) >= book.entries.size:
        raise OracleCorruption(f"quantization code outside [0, {book.entries.size})")
    u = book.entries[c]
    if not u.all():
        raise OracleCorruption("code has no codebook entry (zero frequency at build time)")
    return u


_BATCH = 1 << 20


def deflate(units, chunk):
    """huffman.py:219-269: codewords concatenated MSB-first, every chunk of
    `chunk` codes starts on a byte boundary and is zero-padded to a byte.
    Returns (chunk_bits u32, payload bytes)."""
    if chunk < 1:
        raise OracleError("chunk_size must be >= 1")
    u = np.asarray(units)
    n = u.size
    if n == 0:
        return np.zeros(0, np.uint32), b""
    unit = u.dtype.itemsize * 8
    u64 = u.astype(np.uint64).reshape(-1)
    w = (u64 >> np.uint64(unit - 8)).astype(np.int64)
    if int(w.min()) < 1:
        raise OracleCorruption("packed unit with zero bitwidth")
    cw = u64 & np.uint64((1 << (unit - 8)) - 1)
    nch = -(-n // chunk)
    # bits per chunk via a segmented sum
    starts = np.arange(nch, dtype=np.int64) * chunk
    bits = np.add.reduceat(w, starts).astype(np.int64)
    nbytes = (bits + 7) >> 3
    byte_off = np.concatenate(([0], np.cumsum(nbytes)))
    out = np.zeros(int(byte_off[-1]) * 8, dtype=np.uint8)
    # bit offset of each code inside its own chunk
    cum = np.cumsum(w)
    excl = cum - w
    chunk_of = np.arange(n, dtype=np.int64) // chunk
    first_excl = excl[starts]
    pos = byte_off[chunk_of] * 8 + (excl - first_excl[chunk_of])
    for lo in range(0, n, _BATCH):
        hi = min(n, lo + _BATCH)
        ww = w[lo:hi]
        k = np.repeat(np.arange(hi - lo, dtype=np.int64), ww)     # owning code of each bit
        first_bit = np.cumsum(ww) - ww
        j = np.arange(int(ww.sum()), dtype=np.int64) - first_bit[k]  # bit index inside the code
        shift = (ww[k] - 1 - j).astype(np.uint64)
        out[pos[lo:hi][k] + j] = ((cw[lo:hi][k] >> shift) & np.uint64(1)).astype(np.uint8)
    return bits.astype(np.uint32), np.packbits(out).tobytes()


def _limits(book):
    """huffman.py:272-279: left-aligned exclusive upper bound per width."""
    mx = book.max_bw
    cnt = np.diff(book.offsets)
    lim = np.zeros(mx, dtype=np.uint64)
    for b in range(1, mx + 1):
        lim[b - 1] = (int(book.first[b]) + int(cnt[b])) << (mx - b)
    return lim


def inflate(chunk_bits, payload, chunk, book, n, workers=1):
    """huffman.py:311-356 (+ lockstep decode :282-308): the same checks and
    messages, the same 64-bit big-endian peek window over payload+8 zeros."""
    bits = np.asarray(chunk_bits, dtype=np.int64)
    nch = bits.size
    if n == 0:
        if nch or payload:
            raise OracleCorruption("nonempty stream for zero codes")
        return np.empty(0, np.uint32)
    if chunk < 1 or nch != -(-n // chunk):
        raise OracleCorruption(f"{nch} chunks inconsistent with {n} codes of chunk size {chunk}")
    byte_off = np.concatenate(([0], np.cumsum((bits + 7) >> 3)))
    if int(byte_off[-1]) != len(payload):
        raise OracleCorruption(
            f"payload is {len(payload)} bytes, chunk lengths require {int(byte_off[-1])}")
    per = np.full(nch, chunk, dtype=np.int64)
    per[-1] = n - (nch - 1) * chunk
    buf = np.frombuffer(bytes(payload) + bytes(8), dtype=np.uint8)
    lim = _limits(book)
    mx = book.max_bw
    out = np.empty(n, dtype=np.uint32)
    eight = np.arange(8, dtype=np.int64)

    def run(c0, c1):
        m = c1 - c0
        pos = np.zeros(m, dtype=np.int64)
        base = byte_off[c0:c1] * 8
        budget = bits[c0:c1]
        for k in range(int(per[c0:c1].max())):
            act = m if per[c1 - 1] > k else m - 1
            g = base[:act] + pos[:act]
            win = buf[(g >> 3)[:, None] + eight].view(">u8").reshape(-1)
            peek = (win << (g & 7).astype(np.uint64)) >> np.uint64(64 - mx)
            b = np.searchsorted(lim, peek, side="right").astype(np.int64) + 1
            if int(b.max()) > mx:
                raise OracleCorruption("bit pattern matches no codeword bitwidth")
            npos = pos[:act] + b
            if np.any(npos > budget[:act]):
                raise OracleCorruption("chunk bit budget exhausted mid-codeword")
            top = peek >> (np.uint64(mx) - b.astype(np.uint64))
            s = book.offsets[b] + (top - book.first[b]).astype(np.int64)
            out[(np.arange(c0, c0 + act, dtype=np.int64)) * chunk + k] = book.symbols[s]
            pos[:act] = npos
        if np.any(pos != budget):
            raise OracleCorruption("decoded bits disagree with recorded chunk length")

    w = max(1, min(int(workers or 1), nch))
    if w == 1:
        run(0, nch)
    else:
        cuts = np.linspace(0, nch, w + 1, dtype=np.int64)
        with ThreadPoolExecutor(max_workers=w) as ex:
            futs = [ex.submit(run, int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
            for f in futs:
                f.result()
    return out


# --------------------------------------------------------------------------
# L3 archive  (archive.py:96-246)
# --------------------------------------------------------------------------

def pack_archive(dims, dtype_code, eb_mode, eb_resolved, eb_specified, cap, block,
                 chunk, bitwidths, out_idx, out_val, chunk_bits, payload):
    """serialize (archive.py:96-140): header then bitwidths, interleaved
    (u64 idx, f64 value) outliers, u32 chunk bits, payload."""
    bw = np.ascontiguousarray(np.asarray(bitwidths, dtype=np.uint8))
    nd = len(dims)
    d3 = tuple(dims) + (1,) * (3 - nd)
    b3 = tuple(block) + (1,) * (3 - nd)
    mx = int(bw.max())
    if mx == 0:
        raise OracleError("bitwidth table has no present symbols")
    hdr = HEADER.pack(MAGIC, 1, dtype_code, nd, eb_mode, *d3, float(eb_resolved),
                      float(eb_specified), cap, *b3, chunk, unit_width(mx),
                      len(out_idx), len(chunk_bits), len(payload))
    rec = np.empty(len(out_idx), dtype=[("i", "<u8"), ("v", "<f8")])
    rec["i"] = out_idx
    rec["v"] = out_val
    return b"".join([hdr, bw.tobytes(), rec.tobytes(),
                     np.asarray(chunk_bits, dtype="<u4").tobytes(), bytes(payload)])


@dataclass
class Parsed:
    dims: tuple
    dtype_code: int
    eb_mode: int
    eb_resolved: float
    eb_specified: float
    cap: int
    block: tuple
    chunk: int
    unit: int
    bitwidths: np.ndarray
    out_idx: np.ndarray
    out_val: np.ndarray
    chunk_bits: np.ndarray
    payload: bytes


def unpack_archive(buf):
    """parse_header + deserialize (archive.py:143-246), same check order."""
    if len(buf) < HEADER_SIZE:
        raise OracleFormatError(f"short read: {len(buf)} bytes, header needs {HEADER_SIZE}")
    (magic, ver, dt, nd, mode, d0, d1, d2, ebr, ebs, cap, b0, b1, b2, chunk, unit,
     nout, nch, pbytes) = HEADER.unpack_from(buf, 0)
    if magic != MAGIC:
        raise OracleFormatError(f"bad magic {magic!r}")
    if ver != 1:
        raise OracleFormatError(f"unsupported version {ver}")
    if dt not in (0, 1):
        raise OracleFormatError(f"unsupported dtype code {dt}")
    if not 1 <= nd <= 3:
        raise OracleFormatError(f"unsupported rank {nd}")
    if mode not in (0, 1):
        raise OracleFormatError(f"unknown error-bound mode {mode}")
    if unit not in (32, 64):
        raise OracleFormatError(f"unsupported unit width {unit}")
    dims = (d0, d1, d2)[:nd]
    n = math.prod(dims)
    if n <= 0:
        raise OracleFormatError("dims product must be positive")
    if cap < 4 or cap > 65536 or cap & (cap - 1):
        raise OracleFormatError(f"cap {cap} is not a power of two in [4, 65536]")
    if not ebr > 0:
        raise OracleFormatError("resolved error bound must be positive")
    if chunk < 1:
        raise OracleFormatError("chunk size must be >= 1")
    total = HEADER_SIZE + cap + 16 * nout + 4 * nch + pbytes
    if len(buf) < total:
        raise OracleFormatError(f"short read: {len(buf)} bytes, header promises {total}")
    if len(buf) > total:
        raise OracleFormatError(f"{len(buf) - total} trailing bytes after the archive")
    o = HEADER_SIZE
    bw = np.frombuffer(buf, np.uint8, cap, o).copy()
    o += cap
    rec = np.frombuffer(buf, [("i", "<u8"), ("v", "<f8")], nout, o)
    o += 16 * nout
    cb = np.frombuffer(buf, "<u4", nch, o).astype(np.uint32)
    o += 4 * nch
    payload = bytes(buf[o:o + pbytes])
    w = bw[bw > 0].astype(np.int64)
    if w.size == 0:
        raise OracleFormatError("bitwidth table has no present symbols")
    mx = int(w.max())
    if mx > 56:
        raise OracleFormatError(f"bitwidth {mx} exceeds the supported maximum")
    if w.size >= 2:
        cnt = np.bincount(w)
        if sum(int(c) << (mx - b) for b, c in enumerate(cnt.tolist()) if b) != 1 << mx:
            raise OracleFormatError("bitwidth table violates Kraft equality")
    if unit_width(mx) != unit:
        raise OracleFormatError(f"unit width {unit} disagrees with maximum bitwidth {mx}")
    idx = rec["i"].astype(np.uint64)
    if idx.size:
        if int(idx.max()) >= n:
            raise OracleFormatError("outlier index out of range")
        if np.any(np.diff(idx.astype(np.int64)) <= 0):
            raise OracleFormatError("outlier indices not strictly ascending")
    expect = int(((cb.astype(np.int64) + 7) >> 3).sum())
    if expect != pbytes:
        raise OracleFormatError(f"payload of {pbytes} bytes disagrees with chunk bit lengths "
                                f"({expect} bytes)")
    if nch != -(-n // chunk):
        raise OracleFormatError(f"{nch} chunks inconsistent with {n} points at chunk size {chunk}")
    return Parsed(dims, dt, mode, ebr, ebs, cap, (b0, b1, b2)[:nd], chunk, unit, bw, idx,
                  rec["v"].astype(np.float64), cb, payload)


# --------------------------------------------------------------------------
# L4 pipeline  (pipeline.py:15-58)
# --------------------------------------------------------------------------

def compress(data, dims=None, *, eb, mode="abs", cap=1024, block_shape=None, chunk_size=None):
    """pipeline.compress (pipeline.py:15-39) -> archive bytes."""
    a = np.asarray(data)
    if dims is None:
        dims = a.shape if a.ndim > 1 else (a.size,)
    dims = tuple(int(d) for d in dims)
    if not dims or any(d < 1 for d in dims):
        raise OracleError(f"all extents must be >= 1, got {dims}")
    if a.size != math.prod(dims):
        raise OracleError(f"data has {a.size} values but dims "
                          f"{'x'.join(map(str, dims))} require {math.prod(dims)}")
    vmin, vmax, nonfinite, dt = describe(a)
    if len(dims) > 3:
        raise OracleError(f"rank {len(dims)} fields are not supported (1-3)")
    if mode not in ("abs", "valrel"):
        raise OracleError(f"unknown error-bound mode {mode!r} (use 'abs' or 'valrel')")
    ebr = resolve_eb(mode, eb, vmin, vmax, nonfinite)
    block = tuple(block_shape) if block_shape is not None else DEFAULT_BLOCKS[len(dims)]
    if len(block) != len(dims):
        raise OracleError(f"block_shape rank {len(block)} does not match field rank {len(dims)}")
    if not (ebr > 0 and math.isfinite(ebr)):
        raise OracleError("error bound must be positive and finite")
    if cap < 4 or cap > 65536 or cap & (cap - 1):
        raise OracleError(f"cap must be a power of two in [4, 65536], got {cap}")
    block = tuple(int(b) for b in block)
    if any(b < 1 for b in block):
        raise OracleError(f"all extents must be >= 1, got {block}")
    a = a.astype(dt, copy=False)
    codes, oi, ov = dualquant(a, dims, ebr, cap, block)
    freq = histogram(codes, cap)
    bw = tree_bitwidths(freq)
    book = canonical_book(bw)
    units = encode(codes, book)
    cs = chunk_size or default_chunk_size(codes.size)
    cb, payload = deflate(units, cs)
    return pack_archive(dims, 0 if dt == np.float32 else 1, 0 if mode == "abs" else 1, ebr,
                        eb, cap, block, cs, bw, oi, ov, cb, payload)


def decompress(blob, workers=1):
    """pipeline.decompress / decompress_archive (pipeline.py:42-58)."""
    p = unpack_archive(blob)
    n = math.prod(p.dims)
    book = canonical_book(p.bitwidths)
    codes = inflate(p.chunk_bits, p.payload, p.chunk, book, n, workers=workers)
    validate_quant(codes, p.out_idx, p.out_val, n, p.cap)
    vals = reconstruct(codes, p.out_idx, p.out_val, p.dims, p.eb_resolved, p.cap, p.block)
    return vals.reshape(p.dims).astype(np.float32 if p.dtype_code == 0 else np.float64)


# --------------------------------------------------------------------------
# synthetic fields (synthetic.py:16-88) -- test-data source only
# --------------------------------------------------------------------------

def smooth_field(dims, seed=1, rows=None):
    """synthetic._smooth (synthetic.py:25-35), optionally only rows
    [r0, r1) of axis 0 (bit-identical to slicing the full field)."""
    dims = tuple(int(d) for d in dims)
    rng = np.random.default_rng(seed)
    axes = list(np.ix_(*(np.arange(d, dtype=np.float64) / d for d in dims)))
    if rows is not None:
        axes[0] = axes[0][rows[0]:rows[1]]
    shape = tuple(ax.shape[i] for i, ax in enumerate(axes))
    field = np.zeros(shape)
    for _ in range(6):
        amp = rng.uniform(0.5, 1.0)
        arg = rng.uniform(0.0, 2.0 * math.pi)
        for t in axes:
            arg = arg + rng.uniform(1.0, 4.0) * 2.0 * math.pi * t
        field += amp * np.sin(arg)
    return field
