// inflate.cu -- K5: chunk-parallel canonical Huffman decode (huffman.py:272-356).
//
// The archive fixes the chunking (default_chunk_size, huffman.py:206-212:
// ~1e4-6e4 chunks of 256..65536 codes), too few for a thread per chunk.  A
// warp decodes one chunk in ROUNDS: a round cuts the next stretch of the
// chunk's bits into L <= 32 lane slices of S bits (S ~ 48 codewords at the
// chunk's average code length), so any chunk size runs out of a small,
// bounded shared-memory stage (the round's payload bytes, prefetched with
// cp.async while the previous round decodes).
//
//   phase 1  every lane decodes from its slice start (usually mid-codeword;
//            lane 0 starts on the round's true boundary) to the first
//            codeword start at/after its slice end (its exit), STORING the
//            symbols in a lane-private shared-memory buffer and recording the
//            codeword starts of the first kWin bits of its slice (head mask).
//            It then decodes on into the next slice until one of its codeword
//            starts is also in the next lane's head mask: from that
//            synchronisation point on both paths coincide (decoding is a
//            function of the position), so those tail symbols are the true
//            symbols of the next lane's unsynchronised prefix.
//   phase 2  lane 0 starts on a true boundary; lane l is on the true path if
//            lane l-1 is and l-1 synchronised with it.  The first lane that
//            did not sync redecodes from its predecessor's exit -- rare.
//   copy     a warp scan of the per-lane true-span counts gives output
//            offsets; every lane copies its buffered span out with 16-byte
//            stores.  The last lane's exit is the next round's true start.
//
// Each symbol is decoded once.  The table (shared memory, built by
// decode_prep_kernel from the canonical codebook) is indexed by the next 12
// payload bits and resolves up to three codewords per lookup: their symbols,
// total length and codeword-start mask.  Codewords longer than 12 bits go
// through a second-level table (or, past its budget, a canonical limit
// search).  The bit cursor is a 64-bit register window refilled one word at a
// time from the stage, so a table step's dependency chain is one shared load.
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
// layout of the table block (u32 words): T | L2 (u32[4096]); T holds u64
// entries of up to three codewords (NS = 3) or u128 entries of up to six
// (NS = 6, for streams of short codes: fewer table steps per codeword)
template <int NS>
struct Fmt {
    static constexpr uint32_t kEntryWords = NS == 6 ? 4 : 2;
    static constexpr uint32_t kOffL2 = kEntryWords * kL1Size;
    static constexpr uint32_t kTabWords = kOffL2 + kL2Max;
};
constexpr uint32_t kTabWordsMax = Fmt<6>::kTabWords;

// T entry (NS = 3, u64), len = bits 60-63:
//   len != 0: the greedy decode of the window, up to three codewords:
//             sym0 (0-15) | sym1 (16-31) | sym2 (32-47) | some sym == 0 (48)
//             | codeword starts at offsets 1..11 (49-59; offset 0 implicit)
//             -> n = 1 + popc(starts)
//   len == 0: the first codeword is longer than 12 bits: second-level base
//             (0-15) | extra bits k (16-20) | second level present (21) | no
//             codeword has this prefix (22); neither flag: canonical search
// T entry (NS = 6, u128): words 0-2 = sym0|sym1<<16, sym2|sym3<<16,
//   sym4|sym5<<16; word 3 = meta: len (28-31); len != 0: some sym == 0 (0)
//   | codeword starts at offsets 1..11 (1-11); len == 0: the long-codeword
//   fields of the u64 entry's low word
// L2 entry:  sym << 16 | len
constexpr uint32_t kLongL2 = 1u << 21;
constexpr uint32_t kLongNone = 1u << 22;
constexpr uint32_t kSymInvalid = 0x81;     // long-path result "no codeword": len 1 + flag bit 7

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

// parts 0-3: a quarter of the T windows each; part 4: second-level table;
// part 5: the fallback LUT;
// part -1: everything (both parts compute the shared preliminaries)
__device__ __forceinline__ void dtab_body(const uint64_t* __restrict__ first,
                                          const int64_t* __restrict__ offsets,
                                          const uint32_t* __restrict__ symbols, int max_bw_arg,
                                          const DevStatus* st, uint32_t* __restrict__ tab,
                                          uint32_t* __restrict__ old_lut, int part, int ns) {
    constexpr int kTParts = 4;
    // p0: T windows [w0, w1); pl2: second-level table; plut: fallback LUT
    const bool p0 = part < kTParts, pl2 = part < 0 || part == kTParts, plut = part < 0 || part == kTParts + 1;
    const uint32_t w0 = part >= 0 && part < kTParts ? (uint32_t)part * (kL1Size / kTParts) : 0u;
    const uint32_t w1 = part >= 0 && part < kTParts ? w0 + kL1Size / kTParts : kL1Size;
    __shared__ uint32_t pmax[kL1Size];
    __shared__ uint32_t s_one[kL1Size];   // first codeword of a 12-bit window: sym << 16 | len
    __shared__ uint16_t pbase[kL1Size];   // second-level base, 0xFFFF = none
    __shared__ unsigned long long s_first[34];
    __shared__ long long s_off[35];
    const int mx = max_bw_arg > 0 ? max_bw_arg : (int)st->max_bw;
    const uint32_t offl2 = ns == 6 ? Fmt<6>::kOffL2 : Fmt<3>::kOffL2;
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
        for (uint32_t i = threadIdx.x; i < kL2Max; i += blockDim.x) tab[offl2 + i] = kSymInvalid;
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
    // T: greedy decode of each 12-bit window (<= ns codewords), one lookup per codeword
    for (uint32_t i = w0 + threadIdx.x; p0 && i < w1; i += blockDim.x) {
        uint32_t o = 0, m = 0, starts = 0, zero = 0, sym[6] = {0, 0, 0, 0, 0, 0};
        while (o < (uint32_t)kL1 && m < (uint32_t)ns) {
            const uint32_t one = s_one[swz12((i << o) & (kL1Size - 1))];
            const uint32_t b = one & 63u;
            if (!b || b > kL1 - o) break;
            sym[m] = one >> 16;
            zero |= sym[m] == 0;
            starts |= 1u << o;
            m++;
            o += b;
        }
        // long entries: second-level base | extra bits | flags (no flag: canonical search)
        const uint32_t longe = pmax[i] ? (pbase[i] != 0xFFFF ? (pbase[i] | ((pmax[i] - kL1) << 16) | kLongL2) : 0u)
                                       : kLongNone;
        if (ns == 6) {
            uint4 e;
            e.x = sym[0] | (sym[1] << 16);
            e.y = sym[2] | (sym[3] << 16);
            e.z = sym[4] | (sym[5] << 16);
            e.w = m ? (zero | (starts & 0xFFEu) | (o << 28)) : longe;
            reinterpret_cast<uint4*>(tab)[i] = e;
        } else {
            const unsigned long long e =
                m ? ((unsigned long long)sym[0] | ((unsigned long long)sym[1] << 16) |
                     ((unsigned long long)sym[2] << 32) | ((unsigned long long)zero << 48) |
                     ((unsigned long long)(starts >> 1) << 49) | ((unsigned long long)o << 60))
                  : (unsigned long long)longe;
            reinterpret_cast<unsigned long long*>(tab)[i] = e;
        }
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
        for (uint32_t j = 0; j < (1u << (k - extra)); j++) tab[offl2 + start + j] = e;
    }
}
// decompress prep in one launch of two clusters: cluster 0 scans the chunk
// byte offsets and clears the hand-back flags and the chunk counter; CTAs of
// cluster 1 build the decode tables (4 x T quarter | L2 | fallback LUT)
__global__ void __cluster_dims__(kScanCtas, 1, 1) __launch_bounds__(1024) decode_prep_kernel(
    const uint64_t* __restrict__ first, const int64_t* __restrict__ offsets,
    const uint32_t* __restrict__ symbols, int max_bw_arg, DevStatus* st, uint32_t* __restrict__ tab,
    uint32_t* __restrict__ old_lut, const uint32_t* __restrict__ chunk_bits, uint64_t C,
    unsigned long long* __restrict__ byte_off, uint8_t* __restrict__ redo, unsigned int* counter, int ns) {
    if (blockIdx.x < kScanCtas) {   // cluster 0: chunk byte offsets, flag clears
        for (uint64_t i = blockIdx.x * 1024ull + threadIdx.x; i < C; i += kScanCtas * 1024ull) redo[i] = 0;
        if (blockIdx.x == 0 && threadIdx.x == 0) *counter = 0;
        cluster_chunk_scan(blockIdx.x, chunk_bits, nullptr, C, byte_off, nullptr, ~0ull, false, 0, st);
    } else if (blockIdx.x < kScanCtas + 6) {   // cluster 1: decode tables
        dtab_body(first, offsets, symbols, max_bw_arg, st, tab, old_lut, (int)(blockIdx.x - kScanCtas), ns);
    }
}

// ---------------------------------------------------------------------------
// decoder
// ---------------------------------------------------------------------------
constexpr uint32_t kSliceMin = 64;         // bits per lane slice
template <int NS>
constexpr uint32_t kSliceMax = NS == 6 ? 160 : 192;   // (NS = 6: short codes, smaller stages)
constexpr uint32_t kTargetCodes = 64;      // codewords per lane slice (sets S from the chunk's bits/code)
constexpr uint32_t kFinalSlices = 48;      // a round whose rest fits 48 slices of S is the chunk's last
// u32 words per lane buffer (odd: distinct banks at equal slots)
template <int NS>
constexpr uint32_t kBufStride = NS == 6 ? 53 : 59;
template <int NS>
constexpr uint32_t kStoreMax = 2 * kBufStride<NS> - NS;   // a step stores NS slots at P <= kStoreMax
// stage of one round: up to kFinalSlices slices + the last exit's overrun + the reader's look-ahead
template <int NS>
constexpr uint32_t kStageUnits = (kFinalSlices * kSliceMax<NS> + 32 + 255) / 128 + 3;   // 16-byte units
constexpr int kDecWarps = 16;
// synchronisation window: the head mask `lo` covers the first 64 bits of a
// slice; kHeadHi adds a second mask over [52, 116).  Measured: the second mask
// cuts lane redecodes ~7x but its per-step cost outweighs them on every
// config, so the tail gives up after 52 bits and the next lane redecodes.
constexpr bool kHeadHi = false;
constexpr uint32_t kHeadBits = 64;
constexpr uint32_t kTailBits = kHeadHi ? 116 : 52;

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
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t addr) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts16(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v) : "memory");
}

struct Dec {
    uint32_t tab_s;           // shared address of the table block
    const uint32_t* symbols;  // global, canonical search only
    int mx;
};

// codeword longer than 12 bits at the top of `peek`, past the second-level
// budget: canonical limit search -> sym << 16 | len
__device__ __noinline__ uint32_t long_search(const uint32_t* symbols, int mx, uint32_t peek) {
    for (int b = kL1 + 1; b <= mx; b++) {
        const unsigned long long top = peek >> (32 - b);
        if (top < sh_lim[b]) {
            if (top < sh_first[b]) return kSymInvalid;
            return (symbols[sh_off[b] + (long long)(top - sh_first[b])] << 16) | (uint32_t)b;
        }
    }
    return kSymInvalid;
}

// symbol words of one table step: NS = 3: sym0 | sym1 << 16, sym2 | zero
// flag << 16; NS = 6: three words of two symbols, then the zero flag (bit 0)
template <int NS>
struct Syms {
    uint32_t w[NS == 6 ? 4 : 2];
    __device__ __forceinline__ uint32_t zero() const { return NS == 6 ? (w[3] & 1u) : (w[1] & 0x10000u); }
    __device__ __forceinline__ uint32_t sym(int q) const {
        return (w[q >> 1] >> (16 * (q & 1))) & 0xFFFFu;
    }
};

// the long-codeword path: second level, no codeword, or canonical search
__device__ __forceinline__ uint32_t long_step(const Dec& d, uint32_t info, uint32_t peek, uint32_t offl2) {
    if (info & kLongL2) {
        const uint32_t k = (info >> 16) & 31u;
        return lds32(d.tab_s + (offl2 + (info & 0xFFFFu) + ((peek << kL1) >> (32 - k))) * 4);
    }
    if (info & kLongNone) return kSymInvalid;
    return long_search(d.symbols, d.mx, peek);
}

// One table step at `peek`: total length, codeword-start mask, symbols.
template <int NS>
__device__ __forceinline__ void dstep(const Dec& d, uint32_t peek, uint32_t& len, uint32_t& mask,
                                      Syms<NS>& sv, uint32_t& bad) {
    uint32_t info;
    if (NS == 6) {
        const uint4 e = lds128(d.tab_s + ((peek >> (32 - kL1)) << 4));
        sv.w[0] = e.x;
        sv.w[1] = e.y;
        sv.w[2] = e.z;
        sv.w[NS == 6 ? 3 : 1] = e.w;
        len = e.w >> 28;
        mask = (e.w & 0xFFEu) | 1u;
        info = e.w;
    } else {
        const unsigned long long e = lds64(d.tab_s + ((peek >> (32 - kL1)) << 3));
        sv.w[0] = (uint32_t)e;
        sv.w[1] = (uint32_t)(e >> 32);
        len = sv.w[1] >> 28;
        mask = ((sv.w[1] >> 16) & 0xFFEu) | 1u;
        info = sv.w[0];
    }
    if (!len) {   // long codeword (or a prefix no codeword has)
        const uint32_t ee = long_step(d, info, peek, Fmt<NS>::kOffL2);
        bad |= ee & 0x80u;
        len = ee & 63u;
        sv.w[0] = ee >> 16;
        if (NS == 6) {
            sv.w[NS == 6 ? 3 : 1] = sv.w[0] ? 0u : 1u;
        } else {
            sv.w[1] = sv.w[0] ? 0u : 0x10000u;
        }
        mask = 1u;
    }
}

// MSB-first bit cursor over a round's stage (raw payload bytes, 16-byte
// aligned): three big-endian words in registers, a funnel shift for the peek
// and a branch-free word advance (the next word is always loaded one step
// ahead of its use).  Positions are bits relative to the chunk's 16-byte base.
struct Cursor {
    uint32_t w0, w1, w2;   // w0 holds the bits [pos - o, pos - o + 32); w2 raw
    uint32_t o;            // bit offset of pos in w0
    uint32_t na;           // shared address of the word after w2
    uint32_t pos;
    __device__ __forceinline__ void seek(uint32_t stage_s, uint32_t origin, uint32_t bit) {
        const uint32_t r = bit - origin;
        const uint32_t a = stage_s + ((r >> 5) << 2);
        w0 = bswap32(lds32(a));
        w1 = bswap32(lds32(a + 4));
        w2 = lds32(a + 8);   // kept raw: swapped when it moves into w1
        na = a + 12;
        o = r & 31u;
        pos = bit;
    }
    __device__ __forceinline__ uint32_t peek() const { return __funnelshift_l(w1, w0, o); }
    // (w2 holds the raw little-endian word: its load latency hides until the window moves again)
    __device__ __forceinline__ void adv(uint32_t n) {   // n <= 32
        o += n;
        pos += n;
        if (o >= 32) {   // predicated: the next word is loaded only when the window moves
            w0 = w1;
            w1 = bswap32(w2);
            w2 = lds32(na);
            na += 4;
            o -= 32;
        }
    }
};

// Lane buffers are interleaved across the warp: slots 2j, 2j+1 of lane l are
// the two halves of word j * 32 + l, so a lane only ever touches its own bank
// (no conflicts whatever the lanes' ordinals).  buf_s = the lane's word 0.
__device__ __forceinline__ uint32_t slot_addr(uint32_t buf_s, uint32_t s) {
    return buf_s + ((s >> 1) << 7) + ((s & 1) << 1);
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// store a step's NS symbol slots at ordinal P (slots past n are
// overwritten by the next step; ordinals past the buffer pile up in its last
// slots and the span is then decoded again by lane_direct): whole slot pairs
// as 32-bit stores, plus a 16-bit store at each odd end
template <int NS>
__device__ __forceinline__ void put(uint32_t buf_s, uint32_t P, const Syms<NS>& sv) {
    const uint32_t Pc = P < kStoreMax<NS> ? P : kStoreMax<NS>;
    const uint32_t w = buf_s + ((Pc >> 1) << 7);   // word of slot Pc
    if (NS == 3) {
        // even: [s0 s1] [s2 .]   odd: [. s0] [s1 s2]
        const bool odd = Pc & 1;
        const uint32_t pair = odd ? __byte_perm(sv.w[0], sv.w[1], 0x5432) : sv.w[0];
        sts32(odd ? w + 128 : w, pair);
        sts16(odd ? w + 2 : w + 128, odd ? sv.w[0] : sv.w[1]);
    } else {
        // even: [s0 s1] [s2 s3] [s4 s5]   odd: [. s0] [s1 s2] [s3 s4] [s5 .]
        if (Pc & 1) {
            sts16(w + 2, sv.w[0]);
            sts32(w + 128, __byte_perm(sv.w[0], sv.w[1], 0x5432));
            sts32(w + 256, __byte_perm(sv.w[1], sv.w[2], 0x5432));
            sts16(w + 384, sv.w[2] >> 16);
        } else {
            sts32(w, sv.w[0]);
            sts32(w + 128, sv.w[1]);
            sts32(w + 256, sv.w[2]);
        }
    }
}

// Phase 1a of one lane: decode from the cursor to the slice end S storing
// symbols at ordinals P.. (lane 0 and restarted lanes start on a true
// boundary), recording the codeword starts of the first 116 bits after A0 in
// two overlapping 64-bit head masks: `lo` = [0, 64), `hi` = [52, 116).  tl = the starts at/after S of the step crossing S (bit
// 0 = S).  One loop: lanes diverge only in its trip count.
template <int NS>
__device__ __forceinline__ void lane_decode(const Dec& d, Cursor& rd, uint32_t A0, uint32_t S, uint32_t buf_s,
                                            uint32_t& P, uint32_t& bad, uint32_t& zf, unsigned long long& lo,
                                            unsigned long long& hi, uint32_t& tl) {
    static_assert(!kHeadHi, "the split loop below records the low head mask only");
    uint32_t len = 0, mask = 0, p = rd.pos;
    Syms<NS> sv;
    unsigned long long l = 0, h = 0;
    // the first kHeadBits of the slice record codeword starts; the rest only decodes
    const uint32_t HB = S - A0 < kHeadBits ? S : A0 + kHeadBits;
    while (rd.pos < HB) {
        p = rd.pos;
        dstep<NS>(d, rd.peek(), len, mask, sv, bad);
        put<NS>(buf_s, P, sv);
        zf |= sv.zero();
        l |= (unsigned long long)mask << (p - A0);
        P += __popc(mask);
        rd.adv(len);
    }
    while (rd.pos < S) {
        p = rd.pos;
        dstep<NS>(d, rd.peek(), len, mask, sv, bad);
        put<NS>(buf_s, P, sv);
        zf |= sv.zero();
        P += __popc(mask);
        rd.adv(len);
    }
    // keep the starts inside the slice (the crossing step may record some past S)
    const uint32_t x = S - A0;
    lo = x < 64 ? l & ((1ull << x) - 1) : l;
    hi = (!kHeadHi || x <= 52) ? 0ull : (x - 52 < 64 ? h & ((1ull << (x - 52)) - 1) : h);
    const uint32_t dS = S - p;   // the last step crossed S when it started < 12 bits before it
    tl = (p < S && dS < 12) ? mask >> dS : 0u;
}

// Phase 1b: from the exit, decode on (ordinals P..) until one of the starts
// at/after S is also in the next lane's head masks (nlo, nhi, relative to S)
// -- the synchronisation point -- or S + 116 / the next lane's slice end S2.  sync_pos = the
// synchronisation point (or the tail's end: a true codeword start as well, on
// a true lane); kt = tail codewords before it.
template <int NS>
__device__ __forceinline__ bool lane_tail(const Dec& d, Cursor& rd, uint32_t S, uint32_t S2, uint32_t tl,
                                          unsigned long long nlo, unsigned long long nhi, uint32_t buf_s,
                                          uint32_t& P, uint32_t& bad, uint32_t& zf, uint32_t& sync_pos,
                                          uint32_t& kt) {
    const unsigned long long h0 = (unsigned long long)tl & nlo;
    if (h0) {   // the crossing step already met the next lane's path
        const uint32_t b = (uint32_t)(__ffsll((long long)h0) - 1);
        sync_pos = S + b;
        kt = __popc(tl & ((1u << b) - 1));
        return true;
    }
    uint32_t n = __popc(tl);
    uint32_t len, mask;
    Syms<NS> sv;
    const uint32_t T = S + kTailBits < S2 ? S + kTailBits : S2;   // the next lane's head masks end at its slice end
    while (rd.pos < T) {
        const uint32_t rt = rd.pos - S;
        dstep<NS>(d, rd.peek(), len, mask, sv, bad);
        put<NS>(buf_s, P, sv);
        zf |= sv.zero();
        const unsigned long long hl = rt < 64 ? ((unsigned long long)mask << rt) & nlo : 0ull;
            const unsigned long long hh = (kHeadHi && rt >= 52) ? ((unsigned long long)mask << (rt - 52)) & nhi : 0ull;
        if (hl | hh) {
            const uint32_t b = hl ? (uint32_t)(__ffsll((long long)hl) - 1) - rt
                                  : (uint32_t)(__ffsll((long long)hh) - 1) + 52 - rt;
            sync_pos = rd.pos + b;
            kt = n + __popc(mask & ((1u << b) - 1));
            return true;
        }
        n += __popc(mask);
        P += __popc(mask);
        rd.adv(len);
    }
    sync_pos = rd.pos;
    kt = n;
    return false;
}

// codeword starts of the head masks below bit x (x < 116)
__device__ __forceinline__ uint32_t head_below(unsigned long long lo, unsigned long long hi, uint32_t x) {
    if (x <= 64) return (uint32_t)__popcll(x == 64 ? lo : (lo & ((1ull << x) - 1)));
    return (uint32_t)__popcll(lo) + (uint32_t)__popcll(hi & ((1ull << (x - 52)) - 1) & ~0xFFFull);
}

__device__ __forceinline__ uint32_t zero_halves(uint32_t w) {
    return ((w & 0xFFFFu) == 0) + ((w >> 16) == 0);
}

// Copy the buffered span (slots [a, a + nl)) to dst: 16-byte stores once dst
// is aligned, 4-byte stores around them.  Zero codes are counted only when
// the lane decoded one (cz).
__device__ __forceinline__ uint32_t copy_out(uint32_t buf_s, uint32_t a, uint32_t nl, uint16_t* dst, bool cz) {
    uint32_t z = 0, s = a, n = nl;
    // slots slot, slot+1 as one word (an odd slot straddles two of the lane's words)
    auto pair = [&](uint32_t slot) -> uint32_t {
        const uint32_t wa = buf_s + ((slot >> 1) << 7);
        const uint32_t w0 = lds32(wa);
        return (slot & 1) ? __byte_perm(w0, lds32(wa + 128), 0x5432) : w0;
    };
    if (n && ((uint32_t)(uintptr_t)dst & 2u)) {   // odd element: one u16
        const uint32_t v = lds16(slot_addr(buf_s, s));
        *dst = (uint16_t)v;
        z += v == 0;
        s++;
        dst++;
        n--;
    }
    while (n >= 2 && ((uint32_t)(uintptr_t)dst & 15u)) {
        const uint32_t w = pair(s);
        *reinterpret_cast<uint32_t*>(dst) = w;
        if (cz) z += zero_halves(w);
        s += 2;
        dst += 2;
        n -= 2;
    }
    for (; n >= 8; n -= 8, s += 8, dst += 8) {
        const uint32_t wa = buf_s + ((s >> 1) << 7);
        uint4 v;
        v.x = lds32(wa);
        v.y = lds32(wa + 128);
        v.z = lds32(wa + 256);
        v.w = lds32(wa + 384);
        if (s & 1) {
            const uint32_t w4 = lds32(wa + 512);
            v.x = __byte_perm(v.x, v.y, 0x5432);
            v.y = __byte_perm(v.y, v.z, 0x5432);
            v.z = __byte_perm(v.z, v.w, 0x5432);
            v.w = __byte_perm(v.w, w4, 0x5432);
        }
        *reinterpret_cast<uint4*>(dst) = v;
        if (cz) z += zero_halves(v.x) + zero_halves(v.y) + zero_halves(v.z) + zero_halves(v.w);
    }
    for (; n >= 2; n -= 2, s += 2, dst += 2) {
        const uint32_t w = pair(s);
        *reinterpret_cast<uint32_t*>(dst) = w;
        if (cz) z += zero_halves(w);
    }
    if (n) {
        const uint32_t v = lds16(slot_addr(buf_s, s));
        *dst = (uint16_t)v;
        z += v == 0;
    }
    return z;
}

// A lane whose true span overflowed its buffer decodes it again straight to
// global memory (rare: a slice of unusually short codewords).
template <int NS>
__device__ __noinline__ uint32_t lane_direct(const Dec& d, uint32_t stage_s, uint32_t origin, uint32_t start,
                                             uint32_t count, uint16_t* dst) {
    Cursor rd;
    rd.seek(stage_s, origin, start);
    uint32_t j = 0, z = 0, bad = 0;
    while (j < count) {
        uint32_t len, mask;
        Syms<NS> sv;
        dstep<NS>(d, rd.peek(), len, mask, sv, bad);
        const uint32_t n = __popc(mask), take = n < count - j ? n : count - j;
        for (uint32_t q = 0; q < take; q++) {
            const uint32_t v = sv.sym((int)q);
            dst[j + q] = (uint16_t)v;
            z += v == 0;
        }
        j += take;
        rd.adv(len);
    }
    return z;
}

// One lane's phase 1 from `start` (ordinal 0): slice, exit, tail.
template <int NS>
__device__ __forceinline__ void lane_phase1(const Dec& d, Cursor& rd, uint32_t stage_s, uint32_t origin,
                                            uint32_t start, uint32_t s0, uint32_t s1, uint32_t s2, bool last,
                                            unsigned long long nlo, unsigned long long nhi, uint32_t buf_s,
                                            uint32_t& P, uint32_t& bad, uint32_t& zf, unsigned long long& lo,
                                            unsigned long long& hi, uint32_t& ex, uint32_t& k, uint32_t& sp,
                                            uint32_t& kt, bool& fwd) {
    uint32_t tl;
    rd.seek(stage_s, origin, start);
    P = 0;
    lane_decode<NS>(d, rd, s0, s1, buf_s, P, bad, zf, lo, hi, tl);
    ex = tl ? s1 + (uint32_t)(__ffs(tl) - 1) : rd.pos;   // first codeword start >= s1
    k = P - (uint32_t)__popc(tl);                        // ordinals before the exit
    fwd = false;
    sp = ex;
    kt = 0;
    if (!last) fwd = lane_tail<NS>(d, rd, s1, s2, tl, nlo, nhi, buf_s, P, bad, zf, sp, kt);
}

// One round: lanes [0, L) decode the slices [s0, s1) of one stretch of a
// chunk (lane 0 from the round's true start); the buffered true spans go to
// out[ob ...].  Returns false to hand the chunk back; next_q = the last
// lane's exit (the next round's true start).
template <int NS>
__device__ __forceinline__ bool decode_round(const Dec& d, uint32_t stage_s, uint32_t origin, uint32_t L,
                                             uint32_t s0, uint32_t s1, uint32_t buf_s, uint16_t* out,
                                             uint32_t& ob, uint32_t cnt, uint32_t& next_q, uint32_t& zeros,
                                             DevStatus* st) {
    const uint32_t lane = lane_id();
    const bool active = lane < L;
    const bool last = lane + 1 == L;
    Cursor rd;
    uint32_t P = 0, bad = 0, zf = 0, tl = 0;
    unsigned long long lo = 0, hi = 0;
    if (active) {
        rd.seek(stage_s, origin, s0);
        lane_decode<NS>(d, rd, s0, s1, buf_s, P, bad, zf, lo, hi, tl);
    }
    const unsigned long long nlo = __shfl_down_sync(kFull, lo, 1);
    const unsigned long long nhi = __shfl_down_sync(kFull, hi, 1);
    const uint32_t s2 = __shfl_down_sync(kFull, s1, 1);
    uint32_t ex = s1, k = 0, sp = s1, kt = 0;
    bool fwd = false;   // this lane's tail met the next lane's path
    if (active) {
        ex = tl ? s1 + (uint32_t)(__ffs(tl) - 1) : rd.pos;
        k = P - (uint32_t)__popc(tl);
        sp = ex;
        if (!last) fwd = lane_tail<NS>(d, rd, s1, s2, tl, nlo, nhi, buf_s, P, bad, zf, sp, kt);
    }
    // phase 2: lane l continues lane l-1's true path from q = sp(l-1): at the
    // synchronisation point (l-1's tail met l's path: l's ordinals before q are
    // dropped), or else at the end of l-1's tail, where l decodes again.  Lanes
    // whose link is broken all redecode at once (failures are rare and
    // isolated); a broken lane 0 or a redecode that fails hands the chunk back.
    bool restarted = false;
    uint32_t rstart = 0;   // where a restarted lane began
    for (uint32_t round = 0;; round++) {
        const bool pfwd = __shfl_up_sync(kFull, fwd, 1);
        const uint32_t psp = __shfl_up_sync(kFull, sp, 1);
        const bool link = !active || (bad == 0 && (lane == 0 || (restarted ? rstart == psp : pfwd)));
        const unsigned broken = __ballot_sync(kFull, !link);
        if (broken == 0) break;
        if ((broken & 1u) || round >= L) return false;
        if (!link) {
            restarted = true;
            rstart = psp;
            bad = 0;
            zf = 0;
            lane_phase1<NS>(d, rd, stage_s, origin, psp, s0, s1, s2, last, nlo, nhi, buf_s, P, bad, zf, lo, hi, ex, k, sp,
                            kt, fwd);
            atomicAdd(&st->pad[0], 1ull);   // diagnostics: lane redecodes (low word)
        }
    }
    // true span: ordinals [a, k) up to the exit, plus the tail up to sp
    const uint32_t psp = __shfl_up_sync(kFull, sp, 1);
    const uint32_t q = lane == 0 ? s0 : psp;
    uint32_t a = 0, nl = 0;
    if (active) {
        if (lane != 0 && !restarted) a = head_below(lo, hi, q - s0);
        nl = k - a;
        if (!last) nl += kt;
    }
    int total;
    const uint32_t o = (uint32_t)warp_excl_scan((int)nl, &total);
    next_q = __shfl_sync(kFull, ex, L - 1);
    if (ob + (uint32_t)total > cnt) return false;
    if (nl) {
        uint16_t* dst = out + ob + o;
        if (a + nl <= kStoreMax<NS>) {
            zeros += copy_out(buf_s, a, nl, dst, zf != 0);
        } else {
            zeros += lane_direct<NS>(d, stage_s, origin, q, nl, dst);
            atomicAdd(&st->pad[0], 1ull << 32);   // diagnostics: buffer overflows (high word)
        }
    }
    ob += (uint32_t)total;
    return true;
}

// issue the cp.async loads of stage units [u0, u0 + units) (chunk-relative
// 16-byte units from cb16) into stage_s; units past the payload read zeros
template <int NS>
__device__ __forceinline__ void stage_issue(uint32_t stage_s, const uint4* payload4, uint64_t n4, uint64_t cb16,
                                            uint32_t u0, uint32_t units) {
    if (units > kStageUnits<NS>) units = kStageUnits<NS>;
    for (uint32_t i = lane_id(); i < units; i += 32) {
        const uint64_t u = cb16 + u0 + i;
        const bool in = u < n4;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(stage_s + 16 * i),
                     "l"(payload4 + (in ? u : 0)), "r"(in ? 16 : 0)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// stage units [first, last] covering a round that starts at q and ends by `end` (bits)
__device__ __forceinline__ void round_units(uint32_t q, uint32_t end, uint32_t& u0, uint32_t& units) {
    u0 = q >> 7;
    units = ((end + 32 + 255) >> 7) - u0 + 1;
}

// slice size: ~target codewords at the chunk's mean code length
template <int NS>
__device__ __forceinline__ uint32_t slice_bits(uint32_t B, uint32_t cnt, uint32_t target) {
    const unsigned long long s = (unsigned long long)target * B / (cnt ? cnt : 1);
    return (uint32_t)(s < kSliceMin ? kSliceMin : (s > kSliceMax<NS> ? kSliceMax<NS> : s));
}

// dynamic shared memory: tables (kTabWords) | per-warp lane buffers | per-warp
// double stage
template <int kWarps, int NS>
__global__ void __launch_bounds__(kWarps * 32, 1) inflate_fast_kernel(
    const uint8_t* __restrict__ payload, uint64_t nwords, const uint32_t* __restrict__ chunk_bits,
    const unsigned long long* __restrict__ byte_off, uint64_t nchunks, uint32_t chunk, uint64_t n,
    const uint64_t* __restrict__ gfirst, const int64_t* __restrict__ goffsets,
    const uint32_t* __restrict__ symbols, const uint32_t* __restrict__ gtab, int max_bw_arg,
    uint16_t* __restrict__ out, uint8_t* __restrict__ redo, unsigned int* __restrict__ next_chunk,
    uint32_t target, DevStatus* st) {
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
        const uint32_t words = mx > kL1 ? Fmt<NS>::kTabWords : Fmt<NS>::kOffL2;   // the second level only for long codes
        for (uint32_t i = threadIdx.x; i < words / 4; i += blockDim.x) dst[i] = __ldg(src + i);
        for (int b = threadIdx.x; b < 34; b += blockDim.x) {
            const bool in = b >= 1 && b <= mx;
            sh_first[b] = in ? gfirst[b] : 0;
            sh_lim[b] = in ? gfirst[b] + (unsigned long long)(goffsets[b + 1] - goffsets[b]) : 0;
        }
        for (int b = threadIdx.x; b < 35; b += blockDim.x) sh_off[b] = b <= mx + 1 ? goffsets[b] : 0;
    }
    __syncthreads();
    Dec d;
    const uint32_t smem_base = (uint32_t)__cvta_generic_to_shared(s_tab);
    // opaque copies: keep the shared addresses in registers instead of
    // re-deriving them from the CTA's shared window inside the loops
    asm volatile("mov.u32 %0, %1;" : "=r"(d.tab_s) : "r"(smem_base));
    d.symbols = symbols;
    d.mx = mx;
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    uint32_t buf_s;
    constexpr uint32_t kTW = Fmt<NS>::kTabWords;
    constexpr uint32_t kBS = kBufStride<NS>, kSU = kStageUnits<NS>;
    asm volatile("mov.u32 %0, %1;" : "=r"(buf_s) : "r"(smem_base + kTW * 4 + (wid * 32 * kBS + lane) * 4));
    const uint32_t stage0 = smem_base + kTW * 4 + kWarps * 32 * kBS * 4 + wid * 2 * kSU * 16;
    const uint4* payload4 = reinterpret_cast<const uint4*>(payload);
    const uint64_t n4 = nwords / 4;
    uint32_t zeros = 0, cur = 0;
    bool have = false;   // stage[cur] holds (in flight) the first round of chunk c

    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(next_chunk, 1u);
    c = __shfl_sync(kFull, c, 0);
    while (c < nchunks) {
        uint32_t cn = 0;   // claim the next chunk early: its first stage is prefetched
        if (lane == 0) cn = atomicAdd(next_chunk, 1u);
        cn = __shfl_sync(kFull, cn, 0);
        const uint32_t B = chunk_bits[c];
        const unsigned long long boff = byte_off[c];
        const uint64_t base = (uint64_t)c * chunk;
        const uint32_t cnt = (uint32_t)umin(chunk, n - base);
        const uint64_t cb16 = boff >> 4;
        const uint32_t sbit = (uint32_t)(boff & 15) * 8;
        const uint32_t E = sbit + B;
        bool good = B != 0 && cnt != 0;
        if (good) {
            const uint32_t S = slice_bits<NS>(B, cnt, target);
            uint32_t q = sbit, ob = 0, u0, units, cz = 0;   // cz: zero codes of this chunk
            round_units(q, (E - q <= kFinalSlices * S) ? E : q + 32 * S, u0, units);
            if (!have) stage_issue<NS>(stage0 + cur * kSU * 16, payload4, n4, cb16, u0, units);
            have = false;
            for (;;) {
                const uint32_t R = E - q;
                const bool fin = R <= kFinalSlices * S;
                uint32_t L, s0, s1, nu0 = 0;
                if (fin) {
                    L = R / kSliceMin;
                    L = L < 1 ? 1 : (L > 32 ? 32 : L);
                    s0 = q + (uint32_t)(((uint64_t)(lane < L ? lane : L) * R) / L);
                    s1 = q + (uint32_t)(((uint64_t)(lane < L ? lane + 1 : L) * R) / L);
                } else {
                    L = 32;
                    s0 = q + lane * S;
                    s1 = s0 + S;
                }
                // prefetch: the next round of this chunk, or the next chunk's first round
                const uint32_t nstage = stage0 + (cur ^ 1) * kSU * 16;
                if (!fin) {
                    const uint32_t nq = q + 32 * S;   // the next round starts in [nq, nq + 32)
                    uint32_t nunits;
                    const uint32_t nend = E - nq <= kFinalSlices * S + 32 ? E : nq + 32 + 32 * S;
                    round_units(nq, nend, nu0, nunits);
                    stage_issue<NS>(nstage, payload4, n4, cb16, nu0, nunits);
                } else if (cn < nchunks) {
                    const unsigned long long nboff = byte_off[cn];
                    const uint32_t nB = chunk_bits[cn];
                    const uint32_t ncnt = (uint32_t)umin(chunk, n - (uint64_t)cn * chunk);
                    const uint32_t nS = slice_bits<NS>(nB, ncnt, target);
                    const uint32_t nsb = (uint32_t)(nboff & 15) * 8;
                    uint32_t a0, au;
                    round_units(nsb, (nB <= kFinalSlices * nS) ? nsb + nB : nsb + 32 * nS, a0, au);
                    stage_issue<NS>(nstage, payload4, n4, nboff >> 4, a0, au);
                    have = true;
                } else {
                    asm volatile("cp.async.commit_group;" ::: "memory");
                }
                asm volatile("cp.async.wait_group 1;" ::: "memory");
                __syncwarp();
                uint32_t next_q = 0;
                good = decode_round<NS>(d, stage0 + cur * kSU * 16, u0 * 128, L, s0, s1, buf_s, out + base, ob,
                                    cnt, next_q, cz, st);
                __syncwarp();   // the stage and the buffers are refilled next
                cur ^= 1;
                if (good && fin) good = next_q == E && ob == cnt;
                if (!good || fin) {
                    if (!good && !fin) {   // the prefetched next round is not needed
                        asm volatile("cp.async.wait_all;" ::: "memory");
                        __syncwarp();
                    }
                    break;
                }
                if (next_q < q + 32 * S || next_q >= E) { good = false; asm volatile("cp.async.wait_all;" ::: "memory"); __syncwarp(); break; }
                q = next_q;
                u0 = nu0;
            }
            if (good) zeros += cz;   // a chunk handed back is counted by the sequential decoder
        }
        if (!good && lane == 0) {
            redo[c] = 1;
            atomicAdd(&st->pad[1], 1ull);       // diagnostics: chunks handed back
        }
        c = cn;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    zeros = __reduce_add_sync(kFull, zeros);
    if (lane == 0 && zeros) atomicAdd(&st->n_zero, (unsigned long long)zeros);
}

}  // namespace

int launch_decode_prep(sdqz_ctx* ctx, const uint64_t* first, const int64_t* offsets,
                       const uint32_t* symbols, int max_bw, uint32_t** tab_out, uint32_t* old_lut,
                       const uint32_t* chunk_bits, uint64_t n_chunks, unsigned long long* byte_off,
                       uint8_t* redo, int ns) {
    int rc = SDQZ_OK;
    uint32_t* tab = scratch_as<uint32_t>(ctx, S_DTAB, kTabWordsMax, &rc);
    unsigned int* counter = scratch_as<unsigned int>(ctx, S_COUNTER, 4, &rc);
    if (!tab || !counter) return rc;
    decode_prep_kernel<<<2 * kScanCtas, 1024, 0, ctx->stream>>>(first, offsets, symbols, max_bw, ctx->d_status, tab,
                                                                old_lut, chunk_bits, n_chunks, byte_off, redo,
                                                                counter, ns);
    SDQZ_LAUNCHED_NAMED(ctx, "decode_prep_kernel");
    *tab_out = tab;
    return SDQZ_OK;
}

// codewords per lane slice (SDQZ_DEC_TARGET overrides, for tuning)
static uint32_t dec_target() {
    static const uint32_t t = [] {
        const char* e = getenv("SDQZ_DEC_TARGET");
        const int v = e ? atoi(e) : 0;
        return (uint32_t)(v >= 8 && v <= 200 ? v : kTargetCodes);
    }();
    return t;
}

template <int kW, int NS>
static void launch_inflate_ns(sdqz_ctx* ctx, const uint8_t* payload, uint64_t nwords,
                              const uint32_t* chunk_bits, const unsigned long long* byte_off,
                              uint64_t n_chunks, uint32_t chunk, uint64_t n, const uint64_t* first,
                              const int64_t* offsets, const uint32_t* symbols, const uint32_t* tab,
                              int max_bw, uint16_t* codes, uint8_t* redo, unsigned int* counter) {
    constexpr size_t smem = (size_t)Fmt<NS>::kTabWords * 4 + (size_t)kW * 32 * kBufStride<NS> * 4 +
                            (size_t)kW * 2 * kStageUnits<NS> * 16 + 16;
    static_assert(smem <= 227 * 1024, "decoder shared memory");
    ensure_smem(ctx, (const void*)inflate_fast_kernel<kW, NS>, smem);
    uint64_t grid = ceil_div(n_chunks, kW);
    if (grid > (uint64_t)ctx->num_sms) grid = ctx->num_sms;
    if (grid < 1) grid = 1;
    inflate_fast_kernel<kW, NS><<<(unsigned)grid, kW * 32, smem, ctx->stream>>>(
        payload, nwords, chunk_bits, byte_off, n_chunks, chunk, n, first, offsets, symbols, tab, max_bw, codes,
        redo, counter, dec_target(), ctx->d_status);
}

// symbols per table step: 6 (u128 entries) for streams of short codes, where
// a 12-bit window usually holds more than three codewords (large config -11%
// decode time), 3 (u64 entries) otherwise (Hurricane, 3.3 bits/code: 5% faster
// than 6); SDQZ_DEC_NS=3|6 overrides (tests keep both paths exact)
int decode_ns(uint64_t payload_bytes, uint64_t n) {
    static const int forced = [] {
        const char* e = getenv("SDQZ_DEC_NS");
        return e ? atoi(e) : 0;
    }();
    if (forced == 3 || forced == 6) return forced;
    return 8 * payload_bytes <= 11 * n / 4 ? 6 : 3;   // <= 2.75 bits per code
}

int launch_inflate_fast(sdqz_ctx* ctx, const uint8_t* payload, uint64_t nwords,
                        const uint32_t* chunk_bits, const unsigned long long* byte_off,
                        uint64_t n_chunks, uint32_t chunk, uint64_t n, const uint64_t* first,
                        const int64_t* offsets, const uint32_t* symbols, const uint32_t* tab,
                        int max_bw, uint16_t* codes, uint8_t* redo, int ns) {
    int rc = SDQZ_OK;
    unsigned int* counter = scratch_as<unsigned int>(ctx, S_COUNTER, 4, &rc);   // cleared by the prep kernel
    if (!counter) return rc;
    if (ns == 6)
        launch_inflate_ns<kDecWarps, 6>(ctx, payload, nwords, chunk_bits, byte_off, n_chunks, chunk, n, first,
                                         offsets, symbols, tab, max_bw, codes, redo, counter);
    else
        launch_inflate_ns<kDecWarps, 3>(ctx, payload, nwords, chunk_bits, byte_off, n_chunks, chunk, n, first,
                                        offsets, symbols, tab, max_bw, codes, redo, counter);
    SDQZ_LAUNCHED_NAMED(ctx, "inflate_fast_kernel");
    return SDQZ_OK;
}

}  // namespace sdqz
