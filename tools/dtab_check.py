"""Diagnostics: the device decode table vs a host restatement."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2007_09625_b200 as S
from paper_2007_09625_b200 import _lib
from oracle import sdqz_oracle as O
sys.path.insert(0, "/tmp")

def host_tab(book, cap):
    mx = book.max_bw; first = [int(x) for x in book.first] + [0] * 60
    offs = [int(x) for x in book.offsets]; offs = offs + [offs[-1]] * 60
    lim = [first[b] + (offs[b + 1] - offs[b]) if b <= mx else 0 for b in range(60)]
    def canon(peek, m):
        for b in range(1, m + 1):
            top = peek >> (64 - b)
            if top < lim[b]:
                return b, int(book.symbols[offs[b] + top - first[b]])
        return 0, 0
    sw = 10 if cap <= 1024 else (12 if cap <= 4096 else 16); nm = {10: 5, 12: 4, 16: 3}[sw]
    out = np.zeros(4096, np.uint64)
    for i in range(4096):
        o = k = L1 = 0; e = 0
        while k < nm and o < 12:
            b, s = canon(((i << o) & 0xFFF) << 52, min(12 - o, mx))
            if not b or (k > 0 and s == 0): break
            e |= s << (k * sw); L1 = b if k == 0 else L1; o += b; k += 1
        out[i] = (e | (o << 50) | (k << 54) | (L1 << 57)) if k else 0
    return out

for dims in ((24, 40, 56), (100, 500, 500)):
    f = S.generate_field("smooth", dims, seed=1).astype(np.float32)
    dev = S.compress_device(torch.from_numpy(f).cuda(), eb=1e-4, mode="valrel")
    S.decompress_device(dev)
    ctx = _lib.context()
    tab = np.zeros(4096, np.uint64)
    ctx.call("sdqz_debug_read", 22, ctypes.c_void_p(tab.ctypes.data), tab.nbytes)
    cnt = (_lib.c_uint64 * 3)()
    ctx.lib.sdqz_debug_counters(ctx.h, cnt, 3)
    p = O.unpack_archive(dev.to_bytes())
    book = O.canonical_book(p.bitwidths)
    want = host_tab(book, p.cap)
    n_dev = (tab >> np.uint64(54)) & np.uint64(7)
    n_host = (want >> np.uint64(54)) & np.uint64(7)
    print(dims, "max_bw", book.max_bw, "equal", np.array_equal(tab, want), "dev n=0:", int((n_dev == 0).sum()),
          "host n=0:", int((n_host == 0).sum()), "counters", list(cnt))
    bad = np.flatnonzero(tab != want)[:5]
    for i in bad:
        print(hex(i), hex(int(tab[i])), hex(int(want[i])))
