// inflate.cu -- K5: chunk-parallel canonical Huffman decode (huffman.py:272-356).
//
// The archive fixes the chunking (default_chunk_size, huffman.py:206-212:
// ~1e4-6e4 chunks), too few for a thread per chunk.  A warp decodes one chunk:
// its bit range is cut into L <= 32 equal lane slices (>= kSliceMin bits).
//
//   phase 1  every lane decodes from its slice start (usually mid-codeword)
//            to the first codeword start at/after its slice end (its exit),
//            counting codewords and recording the codeword starts of the first
//            kWin bits of its slice (head mask).  It then decodes on into the
//            next slice until one of its codeword starts is also in the next
//            lane's head mask: from that synchronisation point on both paths
//            coincide (decoding is a function of the position).
//   phase 2  lane 0 starts on a true boundary; lane l is on the true path if
//            lane l-1 is and l-1 synchronised with it.  The first lane that
//            did not sync redecodes from its predecessor's exit (a true
//            boundary) -- rare with a 128-bit window.
//   phase 3  a warp scan of the per-lane true-span symbol counts gives output
//            offsets and every lane decodes its span again, storing codes.
//
// Tables (shared memory, built once per call by dtab_kernel from the
// canonical codebook) are indexed by the next 12 payload bits and resolve
// SEVERAL codewords per lookup: T1 gives the total length, count and the
// codeword-start mask of the greedy decode of the 12-bit window (phase 1
// needs no symbols); T3 gives up to three symbols with their cumulative
// lengths (phase 3).  Codewords longer than 12 bits go through a second-level
// table (or, past its budget, a canonical limit search).  With ~2-4 bits per
// code this decodes ~3 codewords per table step.
//
// Chunks whose codes exceed 32 bits, or whose decode fails any check, are
// handed to the sequential decoder (huffman.cu inflate_kernel), which
// reproduces the reference's exact error semantics.
#include "kernels.cuh"
#include "scan.cuh"

namespace sdqz {

namespace {

constexpr int kL1 = 12;                    // table index bits
constexpr uint32_t kL1Size = 1u << kL1;
constexpr uint32_t kL2Max = 4096;          // second-level entries (long codes)
constexpr uint32_t kSliceMin = 64;         // bits per lane slice (short chunks keep more lanes busy)
constexpr uint32_t kWin = 128;             // synchronisation window (bits)
// layout of the table block (u32 words): T1 | L2 | T3 (u64)
constexpr uint32_t kOffL2 = kL1Size;
constexpr uint32_t kOffT3 = kL1Size + kL2Max;
constexpr uint32_t kTabWords = kOffT3 + 2 * kL1Size;

// T1 entry:  len (0-3) | count (4-7) | codeword-start mask (8-19) | invalid (20)
//            count 0 = first codeword longer than 12 bits (or invalid)
// T3 entry:  sym0 (0-15) | sym1 (16-31) | sym2 (32-47) | n (48-49) | len1 (50-53)
//            | len12 (54-57) | len123 (58-61) | zeros (62-63)
//            n 0 = long: bits 0-11 second-level base, 12-16 extra bits k,
//            17 second level present, 18 invalid
// L2 entry:  sym << 16 | len
constexpr uint32_t kT1Invalid = 1u << 20;
constexpr uint32_t kLongInvalid = 0x81;    // len 1 + flag (sym|len form)

// ---------------------------------------------------------------------------
// decode tables: one CTA
// ---------------------------------------------------------------------------
// s_one is stored swizzled: the greedy decode reads window (i << o) mod 2^12,
// whose low o bits are zero for every lane, so a plain layout puts a warp's
// reads in one bank for o >= 5; XOR-folding the high bits into the bank bits
// spreads them (conflict-free up to o = 7).
__device__ __forceinline__ uint32_t swz12(uint32_t w) {
    const uint32_t h = w >> 5;
    return w ^ ((h ^ (h >> 5)) & 31u);
}

// parts 0-3: a quarter of the T1/T3 windows each; part 4: second-level table;
// part 5: the fallback LUT;
// part -1: everything (both parts compute the shared preliminaries)
__device__ __forceinline__ void dtab_body(const uint64_t* __restrict__ first,
                                          const int64_t* __restrict__ offsets,
                                          const uint32_t* __restrict__ symbols, int max_bw_arg,
                                          const DevStatus* st, uint32_t* __restrict__ tab,
                                          uint32_t* __restrict__ old_lut, int part) {
    constexpr int kT13Parts = 4;
    // p0: T1/T3 windows [w0, w1); pl2: second-level table; plut: fallback LUT
    const bool p0 = part < kT13Parts, pl2 = part < 0 || part == kT13Parts, plut = part < 0 || part == kT13Parts + 1;
    const uint32_t w0 = part >= 0 && part < kT13Parts ? (uint32_t)part * (kL1Size / kT13Parts) : 0u;
    const uint32_t w1 = part >= 0 && part < kT13Parts ? w0 + kL1Size / kT13Parts : kL1Size;
    __shared__ uint32_t pmax[kL1Size];
    __shared__ uint32_t s_one[kL1Size];   // first codeword of a 12-bit window: sym << 16 | len
    __shared__ uint16_t pbase[kL1Size];   // second-level base, 0xFFFF = none
    __shared__ unsigned long long s_first[34];
    __shared__ long long s_off[35];
    const int mx = max_bw_arg > 0 ? max_bw_arg : (int)st->max_bw;
    if (mx < 1 || mx > kMaxBw) return;
    if (mx > 32) {   // 64-bit codes: only the sequential decoder's table (lut_kernel's rule)
        if (!old_lut || !plut) return;
        const long long ns = offsets[mx + 1];
        for (uint32_t i = threadIdx.x; i < (1u << kLutBits); i += blockDim.x) {
            uint32_t e = 0;
            bool found = false;
            for (int b = 1; b <= kLutBits && !found; b++) {
                const unsigned long long top = i >> (kLutBits - b);
                const unsigned long long cnt = (unsigned long long)(offsets[b + 1] - offsets[b]);
                if (top >= first[b] && top < first[b] + cnt) {
                    long long idx = offsets[b] + (long long)(top - first[b]);
                    if (idx >= ns) idx = ns ? ns - 1 : 0;
                    e = (symbols[idx] & 0xFFFF) | ((uint32_t)b << 16);
                    found = true;
                }
            }
            if (!found) {
                const unsigned long long pmin = (unsigned long long)i << (mx - kLutBits);
                uint32_t b0 = (uint32_t)mx + 1;
                for (int b = kLutBits + 1; b <= mx; b++) {
                    const unsigned long long cnt = (unsigned long long)(offsets[b + 1] - offsets[b]);
                    if (pmin < ((first[b] + cnt) << (mx - b))) { b0 = (uint32_t)b; break; }
                }
                e = b0;
            }
            old_lut[i] = e;
        }
        return;
    }
    for (int b = threadIdx.x; b < 34; b += blockDim.x) s_first[b] = b <= mx ? first[b] : 0;
    for (int b = threadIdx.x; b < 35; b += blockDim.x) s_off[b] = b <= mx + 1 ? offsets[b] : offsets[mx + 1];
    for (uint32_t i = threadIdx.x; i < kL1Size; i += blockDim.x) pmax[i] = 0;
    if (pl2)
        for (uint32_t i = threadIdx.x; i < kL2Max; i += blockDim.x) tab[kOffL2 + i] = kLongInvalid;
    __syncthreads();
    const long long nsym = s_off[mx + 1];
    // longest code under each 12-bit prefix
    const long long lo = mx > kL1 ? s_off[kL1 + 1] : nsym;
    for (long long i = lo + threadIdx.x; i < nsym; i += blockDim.x) {
        int b = kL1 + 1;
        while (b < mx && i >= s_off[b + 1]) b++;
        const unsigned long long code = s_first[b] + (unsigned long long)(i - s_off[b]);
        atomicMax(&pmax[(uint32_t)(code >> (b - kL1))], (uint32_t)b);
    }
    __syncthreads();
    {   // exclusive scan of the second-level sizes 2^(pmax - 12); prefixes past the
        // budget fall back to the canonical search
        __shared__ uint32_t wsum[32];
        const uint32_t t = threadIdx.x, per = kL1Size / 1024;
        uint32_t sz[per], run = 0;
#pragma unroll
        for (uint32_t j = 0; j < per; j++) {
            const uint32_t m = pmax[t * per + j];
            sz[j] = m ? (1u << (m - kL1)) : 0u;
            run += sz[j];
        }
        uint32_t x = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if ((t & 31) >= (uint32_t)o) x += y;
        }
        if ((t & 31) == 31) wsum[t >> 5] = x;
        __syncthreads();
        if (t < 32) {
            uint32_t v = wsum[t];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, v, o);
                if (t >= (uint32_t)o) v += y;
            }
            wsum[t] = v;
        }
        __syncthreads();
        uint32_t acc = x - run + ((t >> 5) ? wsum[(t >> 5) - 1] : 0u);
#pragma unroll
        for (uint32_t j = 0; j < per; j++) {
            pbase[t * per + j] = (sz[j] && acc + sz[j] <= kL2Max) ? (uint16_t)acc : (uint16_t)0xFFFF;
            acc += sz[j];
        }
    }
    __syncthreads();
    // first codeword of every 12-bit window (0: longer than 12 bits / none)
    for (uint32_t i = threadIdx.x; i < kL1Size; i += blockDim.x) {
        uint32_t e = 0;
        for (int b = 1; b <= kL1 && b <= mx; b++) {
            const unsigned long long top = i >> (kL1 - b);
            const unsigned long long cnt = (unsigned long long)(s_off[b + 1] - s_off[b]);
            if (top >= s_first[b] && top < s_first[b] + cnt) {
                e = (symbols[s_off[b] + (long long)(top - s_first[b])] << 16) | (uint32_t)b;
                break;
            }
        }
        s_one[swz12(i)] = e;
    }
    __syncthreads();
    // the sequential fallback decoder's table (huffman.cu lut_kernel format)
    if (old_lut && plut) {
        const int lb = mx < kLutBits ? mx : kLutBits;
        for (uint32_t i = threadIdx.x; i < (1u << kLutBits); i += blockDim.x) {
            uint32_t e = 0;
            if (i < (1u << lb)) {
                const uint32_t one = s_one[swz12((i << (kL1 - lb)) & (kL1Size - 1))];
                if (one && (int)(one & 63u) <= lb) {
                    e = (one >> 16) | ((one & 63u) << 16);
                } else if (lb == mx) {
                    e = 255u << 16;
                } else {   // longer than the LUT: shortest possible width as the search hint
                    const unsigned long long pmin = (unsigned long long)i << (mx - lb);
                    uint32_t b0 = (uint32_t)mx + 1;
                    for (int b = lb + 1; b <= mx; b++) {
                        const unsigned long long cnt = (unsigned long long)(s_off[b + 1] - s_off[b]);
                        if (pmin < ((s_first[b] + cnt) << (mx - b))) { b0 = (uint32_t)b; break; }
                    }
                    e = b0;
                }
            }
            old_lut[i] = e;
        }
    }
    __syncthreads();
    // T1 / T3: greedy decode of each 12-bit window, one table lookup per codeword
    for (uint32_t i = w0 + threadIdx.x; p0 && i < w1; i += blockDim.x) {
        uint32_t o = 0, m = 0, mask = 0, zeros = 0, sym[3] = {0, 0, 0}, cum[3] = {0, 0, 0};
        while (o < (uint32_t)kL1) {
            const uint32_t one = s_one[swz12((i << o) & (kL1Size - 1))];
            const uint32_t b = one & 63u;
            if (!b || b > kL1 - o) break;
            const uint32_t sv = one >> 16;
            mask |= 1u << o;
            if (m < 3) {
                sym[m] = sv;
                cum[m] = o + b;
                zeros += sv == 0;
            }
            m++;
            o += b;
        }
        uint32_t t1;
        unsigned long long t3;
        if (m) {
            t1 = o | (m << 4) | (mask << 8);
            const uint32_t n3 = m < 3 ? m : 3;
            t3 = (unsigned long long)sym[0] | ((unsigned long long)sym[1] << 16) |
                 ((unsigned long long)sym[2] << 32) | ((unsigned long long)n3 << 48) |
                 ((unsigned long long)cum[0] << 50) | ((unsigned long long)cum[n3 > 1 ? 1 : 0] << 54) |
                 ((unsigned long long)cum[n3 - 1] << 58) | ((unsigned long long)zeros << 62);
        } else if (pmax[i]) {   // the codeword is longer than 12 bits
            t1 = 1u << 8;
            t3 = pbase[i] != 0xFFFF ? ((unsigned long long)pbase[i] | ((unsigned long long)(pmax[i] - kL1) << 12) |
                                    (1ull << 17))
                                 : 0ull;
        } else {                // no codeword has this prefix (incomplete code)
            t1 = (1u << 8) | kT1Invalid;
            t3 = 1ull << 18;
        }
        tab[i] = t1;
        tab[kOffT3 + 2 * i] = (uint32_t)t3;
        tab[kOffT3 + 2 * i + 1] = (uint32_t)(t3 >> 32);
    }
    // second-level entries
    for (long long i = lo + threadIdx.x; pl2 && i < nsym; i += blockDim.x) {
        int b = kL1 + 1;
        while (b < mx && i >= s_off[b + 1]) b++;
        const unsigned long long code = s_first[b] + (unsigned long long)(i - s_off[b]);
        const uint32_t p = (uint32_t)(code >> (b - kL1));
        if (pbase[p] == 0xFFFF) continue;
        const uint32_t k = pmax[p] - kL1, extra = (uint32_t)b - kL1;
        const uint32_t low = (uint32_t)(code & ((1ull << extra) - 1));
        const uint32_t start = pbase[p] + (low << (k - extra));
        const uint32_t e = (symbols[i] << 16) | (uint32_t)b;
        for (uint32_t j = 0; j < (1u << (k - extra)); j++) tab[kOffL2 + start + j] = e;
    }
}

__global__ void __launch_bounds__(1024) dtab_kernel(const uint64_t* __restrict__ first,
                                                    const int64_t* __restrict__ offsets,
                                                    const uint32_t* __restrict__ symbols,
                                                    int max_bw_arg, const DevStatus* st,
                                                    uint32_t* __restrict__ tab,
                                                    uint32_t* __restrict__ old_lut) {
    dtab_body(first, offsets, symbols, max_bw_arg, st, tab, old_lut, -1);
}

// decompress prep in one launch of two clusters: cluster 0 scans the chunk
// byte offsets and clears the hand-back flags and the chunk counter; CTAs 0/1
// of cluster 1 build the decode tables (T1/T3 | second level + fallback LUT)
__global__ void __cluster_dims__(kScanCtas, 1, 1) __launch_bounds__(1024) decode_prep_kernel(
    const uint64_t* __restrict__ first, const int64_t* __restrict__ offsets,
    const uint32_t* __restrict__ symbols, int max_bw_arg, DevStatus* st, uint32_t* __restrict__ tab,
    uint32_t* __restrict__ old_lut, const uint32_t* __restrict__ chunk_bits, uint64_t C,
    unsigned long long* __restrict__ byte_off, uint8_t* __restrict__ redo, unsigned int* counter) {
    if (blockIdx.x < kScanCtas) {   // cluster 0: chunk byte offsets, flag clears
        for (uint64_t i = blockIdx.x * 1024ull + threadIdx.x; i < C; i += kScanCtas * 1024ull) redo[i] = 0;
        if (blockIdx.x == 0 && threadIdx.x == 0) *counter = 0;
        cluster_chunk_scan(blockIdx.x, chunk_bits, nullptr, C, byte_off, nullptr, ~0ull, false, 0, st);
    } else if (blockIdx.x < kScanCtas + 6) {   // cluster 1: decode tables (4 x T1/T3 quarter | L2 | LUT)
        dtab_body(first, offsets, symbols, max_bw_arg, st, tab, old_lut, (int)(blockIdx.x - kScanCtas));
    }
}

// ---------------------------------------------------------------------------
// shared decode state
// ---------------------------------------------------------------------------
struct Tabs {
    uint32_t tab_s;           // shared address of the table block
    const uint32_t* symbols;  // global, slow path only
    int mx;
};

__shared__ unsigned long long sh_lim[34];   // (first[b] + count[b]), b <= 32
__shared__ unsigned long long sh_first[34];
__shared__ long long sh_off[35];

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ unsigned long long lds64(uint32_t addr) {
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
}

// codeword longer than 12 bits at the top of `peek`, past the second-level
// budget: canonical limit search -> sym << 16 | len
__device__ __noinline__ uint32_t long_search(const Tabs& t, uint32_t peek) {
    for (int b = kL1 + 1; b <= t.mx; b++) {
        const unsigned long long top = peek >> (32 - b);
        if (top < sh_lim[b]) {
            if (top < sh_first[b]) return kLongInvalid;
            return (t.symbols[sh_off[b] + (long long)(top - sh_first[b])] << 16) | (uint32_t)b;
        }
    }
    return kLongInvalid;
}

// codeword longer than 12 bits at the top of `peek` -> sym << 16 | len, given
// the window's T3 entry (second-level pointer)
__device__ __forceinline__ uint32_t long_entry3(const Tabs& t, uint32_t peek, unsigned long long e3) {
    if (e3 & (1ull << 17)) {
        const uint32_t k = (uint32_t)(e3 >> 12) & 31u;
        const uint32_t idx = (uint32_t)(e3 & 0xFFF) + ((peek << kL1) >> (32 - k));
        return lds32(t.tab_s + (kOffL2 + idx) * 4);
    }
    if (e3 & (1ull << 18)) return kLongInvalid;
    return long_search(t, peek);
}

__device__ __forceinline__ uint32_t long_entry(const Tabs& t, uint32_t peek) {
    return long_entry3(t, peek, lds64(t.tab_s + (kOffT3 + 2 * (peek >> (32 - kL1))) * 4));
}

// one phase-1 table step at `peek`: total length, codeword count, start mask
__device__ __forceinline__ void step1(const Tabs& t, uint32_t peek, uint32_t& len, uint32_t& m,
                                      uint32_t& mask, uint32_t& bad) {
    const uint32_t e = lds32(t.tab_s + ((peek >> (32 - kL1)) << 2));
    if (e & 15u) {
        len = e & 15u;
        m = (e >> 4) & 15u;
        mask = (e >> 8) & 0xFFFu;
    } else {
        const uint32_t ee = (e & kT1Invalid) ? kLongInvalid : long_entry(t, peek);
        bad |= ee & 0x80u;
        len = ee & 63u;
        m = 1;
        mask = 1;
    }
}

// Chunk bits staged in shared memory (big-endian words): the peek is two LDS
// of the words under the bit position and a funnel shift.  Positions are
// absolute bits of the staged window.
struct SmemReader {
    uint32_t base_s;   // shared address of word 0
    uint32_t a;        // bit position
    __device__ __forceinline__ void seek(uint32_t bit) { a = bit; }
    __device__ __forceinline__ uint32_t pos() const { return a; }
    __device__ __forceinline__ uint32_t peek() const {
        const uint32_t wa = base_s + ((a >> 5) << 2);
        return __funnelshift_l(lds32(wa + 4), lds32(wa), a);
    }
    __device__ __forceinline__ void adv(uint32_t n) { a += n; }
};

// Chunk bits read from global memory: two words in registers + one prefetched.
struct GlobalReader {
    const uint32_t* w;    // payload words (chunk-relative)
    uint32_t last;        // last readable word index
    uint32_t wi;          // index of w2
    uint32_t w0, w1, w2;
    uint32_t s, p;
    __device__ __forceinline__ uint32_t ld(uint32_t i) const {
        return bswap32(__ldg(w + (i < last ? i : last)));
    }
    __device__ __forceinline__ void seek(uint32_t bit) {
        const uint32_t i = bit >> 5;
        p = bit;
        s = bit & 31u;
        w0 = ld(i);
        w1 = ld(i + 1);
        wi = i + 2;
        w2 = ld(wi);
    }
    __device__ __forceinline__ uint32_t pos() const { return p; }
    __device__ __forceinline__ uint32_t peek() const { return __funnelshift_l(w1, w0, s); }
    __device__ __forceinline__ void adv(uint32_t n) {   // n <= 32
        const uint32_t s2 = s + n;
        p += n;
        if (s2 >= 32) {
            w0 = w1;
            w1 = w2;
            wi++;
            w2 = ld(wi);
        }
        s = s2 & 31u;
    }
};

// 128-bit (lo, hi) view of `mask` (<= 12 bits) shifted left by r < 128
__device__ __forceinline__ void shl128(uint32_t mask, uint32_t r, unsigned long long& lo,
                                       unsigned long long& hi) {
    const unsigned long long mm = mask;
    lo = r < 64 ? (mm << r) : 0ull;
    hi = r >= 64 ? (mm << (r - 64)) : (r > 52 ? (mm >> (64 - r)) : 0ull);
}

// Phase 1a: decode [A0, H) recording codeword starts relative to A0 in (lo, hi).
// The position only grows, so the 128-bit record splits into three loops with
// plain 64-bit shifts: steps wholly inside lo, steps straddling 64, steps in hi.
template <class Rd>
__device__ __forceinline__ void lane_head(const Tabs& t, Rd& rd, uint32_t A0, uint32_t H,
                                          uint32_t& k, uint32_t& bad, unsigned long long& lo,
                                          unsigned long long& hi) {
    unsigned long long l = 0, h = 0;
    const uint32_t h52 = A0 + 52 < H ? A0 + 52 : H, h64 = A0 + 64 < H ? A0 + 64 : H;
    while (rd.pos() < h52) {   // mask (12 bits) << r stays below bit 64
        uint32_t len, m, mask;
        step1(t, rd.peek(), len, m, mask, bad);
        l |= (unsigned long long)mask << (rd.pos() - A0);
        k += m;
        rd.adv(len);
    }
    while (rd.pos() < h64) {
        uint32_t len, m, mask;
        step1(t, rd.peek(), len, m, mask, bad);
        const uint32_t r = rd.pos() - A0;
        l |= (unsigned long long)mask << r;
        h |= (unsigned long long)mask >> (64 - r);
        k += m;
        rd.adv(len);
    }
    while (rd.pos() < H) {
        uint32_t len, m, mask;
        step1(t, rd.peek(), len, m, mask, bad);
        h |= (unsigned long long)mask << (rd.pos() - A0 - 64);
        k += m;
        rd.adv(len);
    }
    lo = l;
    hi = h;
}

// Phase 1b: decode to the slice end S (counting codewords that start before
// S; exit = first codeword start >= S), then on until a codeword start is in
// the next lane's head mask (nlo, nhi, relative to S) -- the synchronisation
// point -- or T is reached.  kt counts the codewords in [exit, sync).
template <class Rd>
__device__ __forceinline__ bool lane_rest(const Tabs& t, Rd& rd, uint32_t S, uint32_t T,
                                          unsigned long long nlo, unsigned long long nhi,
                                          uint32_t& k, uint32_t& bad, uint32_t& exit_pos,
                                          uint32_t& sync_pos, uint32_t& kt) {
    while (rd.pos() < S) {
        const uint32_t p = rd.pos();
        uint32_t len, m, mask;
        step1(t, rd.peek(), len, m, mask, bad);
        if (p + len <= S) {
            k += m;
            rd.adv(len);
        } else {   // the step crosses S: count starts before S, stop at the first >= S
            const uint32_t d = S - p;
            k += __popc(mask & ((1u << d) - 1));
            const uint32_t mh = mask >> d;
            rd.adv(mh ? d + (uint32_t)__ffs(mh) - 1 : len);
            break;
        }
    }
    exit_pos = rd.pos();
    uint32_t n = 0;
    bool found = false;
    // synchronisation usually comes within a few codewords: steps that start
    // below bit 52 of the window compare against nlo alone
    const uint32_t t52 = S + 52 < T ? S + 52 : T;
    while (rd.pos() < t52) {
        const uint32_t r = rd.pos() - S;
        uint32_t len, m, mask;
        step1(t, rd.peek(), len, m, mask, bad);
        const unsigned long long a = ((unsigned long long)mask << r) & nlo;
        if (a) {
            const uint32_t q = (uint32_t)(__ffsll((long long)a) - 1);
            n += __popc(mask & ((1u << (q - r)) - 1));
            rd.adv(q - r);
            found = true;
            break;
        }
        n += m;
        rd.adv(len);
    }
    while (!found && rd.pos() < T) {
        const uint32_t r = rd.pos() - S;
        uint32_t len, m, mask;
        step1(t, rd.peek(), len, m, mask, bad);
        unsigned long long a, b;
        shl128(mask, r, a, b);
        a &= nlo;
        b &= nhi;
        if (a | b) {
            const uint32_t q = a ? (uint32_t)(__ffsll((long long)a) - 1) : 64u + (uint32_t)(__ffsll((long long)b) - 1);
            n += __popc(mask & ((1u << (q - r)) - 1));
            rd.adv(q - r);
            found = true;
            break;
        }
        n += m;
        rd.adv(len);
    }
    sync_pos = rd.pos();
    kt = n;
    return found;
}

// codeword starts of (lo, hi) below bit r (r <= 128)
__device__ __forceinline__ uint32_t below(unsigned long long lo, unsigned long long hi, uint32_t r) {
    if (r == 0) return 0;
    if (r <= 64) return __popcll(r == 64 ? lo : (lo & ((1ull << r) - 1)));
    return __popcll(lo) + __popcll(r >= 128 ? hi : (hi & ((1ull << (r - 64)) - 1)));
}

// Phase 3 of one lane: `count` codewords from `start` (must end at `end`) into
// dst.  Symbols go through a 16-slot per-lane ring in shared memory; every
// completed 16-byte output vector is written with one store.
template <class Rd>
__device__ __forceinline__ bool lane_store(const Tabs& t, Rd& rd, uint32_t start, uint32_t end,
                                           uint32_t count, uint16_t* dst, uint32_t ring_s,
                                           uint32_t& zeros) {
    rd.seek(start);
    const uint32_t aoff = (uint32_t)((uintptr_t)dst >> 1) & 7u;   // slots before dst in its vector
    uint16_t* const dal = dst - aoff;                               // 16-byte aligned
    uint32_t P = aoff;              // next ring slot (absolute)
    uint32_t nextv = 8;             // slot count at which vector (nextv/8 - 1) completes
    uint32_t j = 0, bad = 0, z = 0;
    while (j < count) {
        const uint32_t peek = rd.peek();
        unsigned long long e3 = lds64(t.tab_s + (kOffT3 + 2 * (peek >> (32 - kL1))) * 4);
        uint32_t n3 = (uint32_t)(e3 >> 48) & 3u, len;
        if (n3 == 0) {   // long codeword (or invalid pattern)
            const uint32_t ee = long_entry3(t, peek, e3);
            bad |= ee & 0x80u;
            len = ee & 63u;
            e3 = ee >> 16;
            n3 = 1;
            z += (ee >> 16) == 0;
        } else if (j + n3 > count) {   // the span ends inside this step
            const uint32_t take = count - j;
            len = take == 1 ? (uint32_t)(e3 >> 50) & 15u : (uint32_t)(e3 >> 54) & 15u;
            z += ((e3 & 0xFFFF) == 0) + (take > 1 && ((e3 >> 16) & 0xFFFF) == 0);
            n3 = take;
        } else {
            len = (uint32_t)(e3 >> 58) & 15u;
            z += (uint32_t)(e3 >> 62);
        }
#pragma unroll
        for (uint32_t q = 0; q < 3; q++) {
            if (q < n3) {
                asm volatile("st.shared.u16 [%0], %1;" ::"r"(ring_s + ((P + q) & 15u) * 2),
                             "h"((unsigned short)(e3 >> (16 * q))));
            }
        }
        P += n3;
        j += n3;
        rd.adv(len);
        if (P >= nextv) {   // vector v = nextv/8 - 1 complete (lane-private ring)
            const uint32_t v = nextv / 8 - 1;
            const uint32_t rs = ring_s + ((8 * v) & 15u) * 2;
            uint4 qv;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(qv.x), "=r"(qv.y) : "r"(rs));
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(qv.z), "=r"(qv.w) : "r"(rs + 8));
            if (v == 0 && aoff) {
                const uint32_t h[8] = {qv.x & 0xFFFF, qv.x >> 16, qv.y & 0xFFFF, qv.y >> 16,
                                       qv.z & 0xFFFF, qv.z >> 16, qv.w & 0xFFFF, qv.w >> 16};
#pragma unroll
                for (uint32_t s = 1; s < 8; s++)
                    if (s >= aoff) dal[s] = (uint16_t)h[s];
            } else {
                *reinterpret_cast<uint4*>(dal + 8 * v) = qv;
            }
            nextv += 8;
        }
    }
    // trailing partial vector
    const uint32_t v = nextv / 8 - 1;
    for (uint32_t s = (v == 0 ? aoff : 0); 8 * v + s < P; s++) {
        unsigned short h;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(ring_s + ((8 * v + s) & 15u) * 2));
        dal[8 * v + s] = h;
    }
    zeros += z;
    return !bad && rd.pos() == end;
}

// Phases 1-3 of one chunk by one warp; positions are absolute bits (the chunk
// occupies [sbit, sbit + B)).  false = hand the chunk back.
template <class Rd>
__device__ __forceinline__ bool decode_chunk(const Tabs& t, Rd rd, uint32_t sbit, uint32_t B,
                                             uint32_t cnt, uint16_t* out, uint32_t ring_s,
                                             uint32_t& zeros, DevStatus* st) {
    const uint32_t lane = lane_id();
    uint32_t L = B / kSliceMin;
    L = L < 1 ? 1 : (L > 32 ? 32 : L);
    const bool active = lane < L;
    const bool last = lane + 1 == L;
    const uint32_t s0 = sbit + (active ? (uint32_t)(((uint64_t)lane * B) / L) : B);
    const uint32_t s1 = sbit + (active ? (uint32_t)(((uint64_t)(lane + 1) * B) / L) : B);
    const uint32_t T = last || !active ? s1 : (s1 + kWin < sbit + B ? s1 + kWin : sbit + B);
    uint32_t k = 0, bad = 0, ex = s1, sp = s1, kt = 0, start = s0;
    unsigned long long lo = 0, hi = 0;
    bool fwd = false;   // this lane's tail met the next lane's path
    if (active) {
        rd.seek(s0);
        // the head window ends >= 12 bits (one table step) before the slice end,
        // so its last step cannot run past S (lane_rest counts exactly to S)
        const uint32_t hend = s1 > s0 + 12 ? (s0 + kWin < s1 - 12 ? s0 + kWin : s1 - 12) : s0;
        lane_head(t, rd, s0, hend, k, bad, lo, hi);
    }
    const unsigned long long nlo = __shfl_down_sync(kFull, lo, 1);
    const unsigned long long nhi = __shfl_down_sync(kFull, hi, 1);
    if (active) fwd = lane_rest(t, rd, s1, T, nlo, nhi, k, bad, ex, sp, kt);
    bool ok = bad == 0;
    // phase 2: lane l is on the true path if lane l-1 is and l-1's tail met it;
    // the first lane that is not redecodes from its predecessor's exit
    bool restarted = lane == 0;
    uint32_t q = s0;   // start of the lane's true span
    for (uint32_t round = 0;; round++) {
        const bool pfwd = __shfl_up_sync(kFull, fwd, 1);
        const uint32_t pe = __shfl_up_sync(kFull, ex, 1);
        const uint32_t psp = __shfl_up_sync(kFull, sp, 1);
        const bool synced = !active || (ok && (restarted || pfwd));
        const unsigned badl = __ballot_sync(kFull, !synced);
        if (badl == 0) {
            if (active && !restarted) q = psp;
            break;
        }
        const uint32_t f = (uint32_t)(__ffs(badl) - 1);
        if (f == 0 || round >= L) return false;
        if (lane == f) {
            restarted = true;
            q = start = pe;
            k = 0;
            bad = 0;
            rd.seek(pe);
            fwd = lane_rest(t, rd, s1, T, nlo, nhi, k, bad, ex, sp, kt);
            ok = bad == 0;
            atomicAdd(&st->pad[0], 1ull);   // diagnostics: lane redecodes
        }
        if (!__shfl_sync(kFull, ok ? 1u : 0u, f)) return false;
    }
    // true-span length of each lane: its codewords from q to its exit, plus its
    // tail codewords up to the next lane's start (if that lane synced on it)
    const bool nrestart = __shfl_down_sync(kFull, restarted, 1);
    const uint32_t nq = __shfl_down_sync(kFull, q, 1);
    const uint32_t last_e = __shfl_sync(kFull, ex, L - 1);
    uint32_t nl = 0;
    if (active) {
        nl = k - (restarted ? 0u : below(lo, hi, q - s0));
        if (!last && !nrestart) nl += kt;
    }
    int total;
    const uint32_t o = (uint32_t)warp_excl_scan((int)nl, &total);
    if (last_e != sbit + B || (uint32_t)total != cnt) return false;
    // phase 3
    bool ok3 = true;
    uint32_t z = 0;
    const uint32_t end = last ? sbit + B : nq;
    if (active && nl) ok3 = lane_store(t, rd, q, end, nl, out + o, ring_s, z);
    if (!__all_sync(kFull, ok3)) return false;
    zeros += z;
    return true;
}

// one CTA per SM shares one copy of the tables: 32 warps, or 24 for chunks of
// >= 16384 codes (longer lane spans: the register budget of 1024-thread CTAs
// is the limit there, and fewer warps leave more staging per warp)
constexpr uint32_t kRingStride = 40;   // 16 u16 slots per lane + 8 bytes: 2-way bank conflicts

// dynamic shared memory: tables (kTabWords) | per-lane rings | one staging
// buffer of `stage_words` words per warp
template <int kWarps>
__global__ void __launch_bounds__(kWarps * 32) inflate_fast_kernel(
    const uint8_t* __restrict__ payload, uint64_t nwords, const uint32_t* __restrict__ chunk_bits,
    const unsigned long long* __restrict__ byte_off, uint64_t nchunks, uint32_t chunk, uint64_t n,
    const uint64_t* __restrict__ gfirst, const int64_t* __restrict__ goffsets,
    const uint32_t* __restrict__ symbols, const uint32_t* __restrict__ gtab, int max_bw_arg,
    uint16_t* __restrict__ out, uint8_t* __restrict__ redo, unsigned int* __restrict__ next_chunk,
    uint32_t stage_words, DevStatus* st) {
    extern __shared__ __align__(16) uint32_t s_tab[];
    const int mx = max_bw_arg > 0 ? max_bw_arg : (int)st->max_bw;
    if (mx < 1 || mx > 32) {   // 64-bit codes: everything goes to the sequential decoder
        for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < nchunks;
             c += (uint64_t)gridDim.x * blockDim.x)
            redo[c] = 1;
        if (blockIdx.x == 0 && threadIdx.x == 0 && nchunks) atomicAdd(&st->pad[1], 1ull);
        return;
    }
    {
        const uint4* src = reinterpret_cast<const uint4*>(gtab);
        uint4* dst = reinterpret_cast<uint4*>(s_tab);
        for (uint32_t i = threadIdx.x; i < kTabWords / 4; i += blockDim.x) dst[i] = __ldg(src + i);
        for (int b = threadIdx.x; b < 34; b += blockDim.x) {
            const bool in = b >= 1 && b <= mx;
            sh_first[b] = in ? gfirst[b] : 0;
            sh_lim[b] = in ? gfirst[b] + (unsigned long long)(goffsets[b + 1] - goffsets[b]) : 0;
        }
        for (int b = threadIdx.x; b < 35; b += blockDim.x) sh_off[b] = b <= mx + 1 ? goffsets[b] : 0;
    }
    __syncthreads();
    Tabs t;
    const uint32_t smem_base = (uint32_t)__cvta_generic_to_shared(s_tab);
    asm volatile("mov.u32 %0, %1;" : "=r"(t.tab_s) : "r"(smem_base));
    t.symbols = symbols;
    t.mx = mx;
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    const uint32_t ring_s = smem_base + kTabWords * 4 + threadIdx.x * kRingStride;
    uint32_t* stage = s_tab + kTabWords + (kWarps * 32 * kRingStride) / 4 + wid * stage_words;
    const uint32_t* words = reinterpret_cast<const uint32_t*>(payload);
    const uint4* words4 = reinterpret_cast<const uint4*>(payload);
    uint32_t zeros_total = 0;

    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(next_chunk, 1u);
    c = __shfl_sync(kFull, c, 0);
    while (c < nchunks) {
        uint32_t cn = 0;   // claim the next chunk early: the atomic's latency hides behind this one
        if (lane == 0) cn = atomicAdd(next_chunk, 1u);
        const uint32_t B = chunk_bits[c];
        const unsigned long long boff = byte_off[c];
        const uint64_t base = (uint64_t)c * chunk;
        const uint32_t cnt = (uint32_t)umin(chunk, n - base);
        // 16-byte aligned window of the payload holding the chunk (+ 2 words of peek slack)
        const uint64_t q0 = boff >> 4;
        const uint32_t sbit = (uint32_t)(boff & 15) * 8;
        const uint32_t nq4 = (uint32_t)(((uint64_t)sbit + B + 63 + 127) >> 7);
        bool good;
        if (nq4 * 4 <= stage_words && (q0 + nq4) * 4 <= nwords) {
            for (uint32_t i = lane; i < nq4; i += 32) {
                const uint4 v = __ldg(words4 + q0 + i);
                reinterpret_cast<uint4*>(stage)[i] =
                    make_uint4(bswap32(v.x), bswap32(v.y), bswap32(v.z), bswap32(v.w));
            }
            __syncwarp();
            SmemReader rd;
            rd.base_s = (uint32_t)__cvta_generic_to_shared(stage);
            good = decode_chunk(t, rd, sbit, B, cnt, out + base, ring_s, zeros_total, st);
            __syncwarp();   // the stage is refilled by the next chunk
        } else {
            const uint64_t wbase = boff >> 2;
            GlobalReader rd;
            rd.w = words + wbase;
            rd.last = (uint32_t)umin(nwords > wbase ? nwords - 1 - wbase : 0, 0xFFFFFFFFull);
            good = decode_chunk(t, rd, (uint32_t)(boff & 3) * 8, B, cnt, out + base, ring_s,
                                zeros_total, st);
        }
        if (!good && lane == 0) {
            redo[c] = 1;
            atomicAdd(&st->pad[1], 1ull);       // diagnostics: chunks handed back
        }
        c = __shfl_sync(kFull, cn, 0);
    }
    zeros_total = __reduce_add_sync(kFull, zeros_total);
    if (lane == 0 && zeros_total) atomicAdd(&st->n_zero, (unsigned long long)zeros_total);
}

}  // namespace

int launch_decode_tables(sdqz_ctx* ctx, const uint64_t* first, const int64_t* offsets,
                         const uint32_t* symbols, int max_bw, uint32_t** tab_out, uint32_t* old_lut) {
    int rc = SDQZ_OK;
    uint32_t* tab = scratch_as<uint32_t>(ctx, S_DTAB, kTabWords, &rc);
    if (!tab) return rc;
    dtab_kernel<<<1, 1024, 0, ctx->stream>>>(first, offsets, symbols, max_bw, ctx->d_status, tab,
                                             old_lut);
    SDQZ_LAUNCHED_NAMED(ctx, "dtab_kernel");
    *tab_out = tab;
    return SDQZ_OK;
}

int launch_decode_prep(sdqz_ctx* ctx, const uint64_t* first, const int64_t* offsets,
                       const uint32_t* symbols, int max_bw, uint32_t** tab_out, uint32_t* old_lut,
                       const uint32_t* chunk_bits, uint64_t n_chunks, unsigned long long* byte_off,
                       uint8_t* redo) {
    int rc = SDQZ_OK;
    uint32_t* tab = scratch_as<uint32_t>(ctx, S_DTAB, kTabWords, &rc);
    unsigned int* counter = scratch_as<unsigned int>(ctx, S_COUNTER, 4, &rc);
    if (!tab || !counter) return rc;
    decode_prep_kernel<<<2 * kScanCtas, 1024, 0, ctx->stream>>>(first, offsets, symbols, max_bw, ctx->d_status, tab,
                                                    old_lut, chunk_bits, n_chunks, byte_off, redo,
                                                    counter);
    SDQZ_LAUNCHED_NAMED(ctx, "decode_prep_kernel");
    *tab_out = tab;
    return SDQZ_OK;
}

template <int kWarps>
void launch_inflate_fast_w(sdqz_ctx* ctx, const uint8_t* payload, uint64_t nwords, const uint32_t* chunk_bits,
                           const unsigned long long* byte_off, uint64_t n_chunks, uint32_t chunk, uint64_t n,
                           const uint64_t* first, const int64_t* offsets, const uint32_t* symbols,
                           const uint32_t* tab, int max_bw, uint16_t* codes, uint8_t* redo, unsigned int* counter) {
    // per-warp staging: room for ~2x the average chunk (bigger chunks read global memory)
    const uint64_t avg = n_chunks ? (nwords * 4) / n_chunks : 0;
    const size_t fixed = (size_t)kTabWords * 4 + (size_t)kWarps * 32 * kRingStride;
    int smem_max = 0;
    cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
    const uint32_t room = (uint32_t)(((size_t)smem_max - 1024 - fixed) / (kWarps * 4)) & ~15u;
    uint32_t stage_words = (uint32_t)umin(((2 * avg + 64) / 4 + 15) & ~15ull, room);
    if (stage_words < 64) stage_words = 64;
    const size_t smem = fixed + (size_t)kWarps * stage_words * 4;
    ensure_smem(ctx, (const void*)inflate_fast_kernel<kWarps>, smem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, inflate_fast_kernel<kWarps>, kWarps * 32, smem);
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = ceil_div(n_chunks, kWarps);
    const uint64_t cap = (uint64_t)ctx->num_sms * per_sm;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    inflate_fast_kernel<kWarps><<<(unsigned)grid, kWarps * 32, smem, ctx->stream>>>(
        payload, nwords, chunk_bits, byte_off, n_chunks, chunk, n, first, offsets, symbols, tab,
        max_bw, codes, redo, counter, stage_words, ctx->d_status);
}

int launch_inflate_fast(sdqz_ctx* ctx, const uint8_t* payload, uint64_t nwords,
                        const uint32_t* chunk_bits, const unsigned long long* byte_off,
                        uint64_t n_chunks, uint32_t chunk, uint64_t n, const uint64_t* first,
                        const int64_t* offsets, const uint32_t* symbols, const uint32_t* tab,
                        int max_bw, uint16_t* codes, uint8_t* redo) {
    int rc = SDQZ_OK;
    unsigned int* counter = scratch_as<unsigned int>(ctx, S_COUNTER, 4, &rc);   // cleared by the prep kernel
    if (!counter) return rc;
    if (chunk >= 16384)
        launch_inflate_fast_w<24>(ctx, payload, nwords, chunk_bits, byte_off, n_chunks, chunk, n, first, offsets,
                                  symbols, tab, max_bw, codes, redo, counter);
    else
        launch_inflate_fast_w<32>(ctx, payload, nwords, chunk_bits, byte_off, n_chunks, chunk, n, first, offsets,
                                  symbols, tab, max_bw, codes, redo, counter);
    SDQZ_LAUNCHED_NAMED(ctx, "inflate_fast_kernel");
    return SDQZ_OK;
}

}  // namespace sdqz
