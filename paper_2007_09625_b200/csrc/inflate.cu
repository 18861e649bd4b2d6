// inflate.cu -- K5: chunk-parallel canonical Huffman decode (huffman.py:272-356).
//
// The archive fixes the chunking (default_chunk_size, huffman.py:206-212:
// ~1e4-6e4 chunks), too few for a thread per chunk.  A warp decodes one chunk:
// its bit range is cut into L <= 32 equal lane slices (>= kSliceMin bits).
//
//   phase 1  every lane decodes from its slice start (usually mid-codeword)
//            to the first codeword boundary at/after its slice end (its exit),
//            counting codewords, and records the codeword boundaries of the
//            first kWin bits of its slice (wa) and of the first kWin bits of
//            the NEXT slice (wb, decoding on past its end).
//   phase 2  lane 0 starts on a true boundary.  Lane l is synchronised with
//            lane l-1 when wa_l & wb_{l-1} != 0: from that first common
//            boundary on both paths coincide (Huffman decoding is a function
//            of the position), so lane l's path is the true path.  Lanes are
//            checked all at once with a ballot; the first unsynchronised lane
//            redecodes from its predecessor's exit (a true boundary) and the
//            ballot is repeated -- at most L rounds, usually one.
//   phase 3  a warp scan of the per-lane true-symbol counts gives output
//            offsets and every lane decodes its true span again, packing codes
//            into 16-byte stores.
//
// Decode step: a 32-bit peek is a funnel shift of two big-endian payload
// words held in registers (a third is prefetched); a 12-bit primary table in
// shared memory resolves codewords <= 12 bits, longer ones go through a
// per-prefix second-level table (also shared; sized 2^(max len under the
// prefix - 12)) or, if that does not fit, a canonical limit search.  Chunks
// whose codes exceed 32 bits, or whose decode fails any check, are handed to
// the sequential decoder (huffman.cu inflate_kernel), which reproduces the
// reference's exact error semantics.
#include "kernels.cuh"

namespace sdqz {

namespace {

constexpr int kL1 = 12;                    // primary table bits
constexpr uint32_t kL1Size = 1u << kL1;
constexpr uint32_t kL2Max = 4096;          // second-level entries
constexpr uint32_t kSliceMin = 192;        // bits per lane slice (> kWin)
constexpr uint32_t kWin = 128;             // synchronisation window (bits)
constexpr uint32_t kTabWords = kL1Size + kL2Max;

// entry: short/full  sym << 16 | len            (len 1..32)
//        second level base << 16 | k << 8 | 0x40 (len field 0, k extra bits)
//        slow         0                          (canonical limit search)
//        invalid      0x80 | 1                   (no codeword: incomplete code)
constexpr uint32_t kInvalid = 0x81;          // len 1 + flag: loops stay bounded

// ---------------------------------------------------------------------------
// decode tables: one CTA builds primary + second-level tables in global memory
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) dtab_kernel(const uint64_t* __restrict__ first,
                                                    const int64_t* __restrict__ offsets,
                                                    const uint32_t* __restrict__ symbols,
                                                    int max_bw_arg, const DevStatus* st,
                                                    uint32_t* __restrict__ tab) {
    __shared__ uint32_t pmax[kL1Size];
    __shared__ uint32_t pbase[kL1Size];
    __shared__ unsigned long long s_first[34];
    __shared__ long long s_off[35];
    const int mx = max_bw_arg > 0 ? max_bw_arg : (int)st->max_bw;
    if (mx < 1 || mx > 32) return;                // > 32: the warp decoder is not used
    for (int b = threadIdx.x; b < 34; b += blockDim.x) s_first[b] = b <= mx ? first[b] : 0;
    for (int b = threadIdx.x; b < 35; b += blockDim.x) s_off[b] = b <= mx + 1 ? offsets[b] : offsets[mx + 1];
    for (uint32_t i = threadIdx.x; i < kL1Size; i += blockDim.x) pmax[i] = 0;
    for (uint32_t i = threadIdx.x; i < kL2Max; i += blockDim.x) tab[kL1Size + i] = kInvalid;
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
            pbase[t * per + j] = (sz[j] && acc + sz[j] <= kL2Max) ? acc : ~0u;
            acc += sz[j];
        }
    }
    __syncthreads();
    // primary entries
    for (uint32_t i = threadIdx.x; i < kL1Size; i += blockDim.x) {
        uint32_t e = kInvalid;
        bool found = false;
        for (int b = 1; b <= kL1 && b <= mx && !found; b++) {
            const unsigned long long top = i >> (kL1 - b);
            const unsigned long long cnt = (unsigned long long)(s_off[b + 1] - s_off[b]);
            if (top >= s_first[b] && top < s_first[b] + cnt) {
                const long long idx = s_off[b] + (long long)(top - s_first[b]);
                e = (symbols[idx] << 16) | (uint32_t)b;
                found = true;
            }
        }
        if (!found && pmax[i]) {
            e = pbase[i] != ~0u ? ((pbase[i] << 16) | ((pmax[i] - kL1) << 8) | 0x40u) : 0u;
        }
        tab[i] = e;
    }
    // second-level entries
    for (long long i = lo + threadIdx.x; i < nsym; i += blockDim.x) {
        int b = kL1 + 1;
        while (b < mx && i >= s_off[b + 1]) b++;
        const unsigned long long code = s_first[b] + (unsigned long long)(i - s_off[b]);
        const uint32_t p = (uint32_t)(code >> (b - kL1));
        if (pbase[p] == ~0u) continue;
        const uint32_t k = pmax[p] - kL1, extra = (uint32_t)b - kL1;
        const uint32_t low = (uint32_t)(code & ((1ull << extra) - 1));
        const uint32_t start = pbase[p] + (low << (k - extra));
        const uint32_t e = (symbols[i] << 16) | (uint32_t)b;
        for (uint32_t j = 0; j < (1u << (k - extra)); j++) tab[kL1Size + start + j] = e;
    }
}

// ---------------------------------------------------------------------------
// shared decode state
// ---------------------------------------------------------------------------
struct Tabs {
    uint32_t tab_s;           // shared address of the tables
    const uint32_t* symbols;  // global, slow path only
    int mx;
};

__shared__ unsigned long long sh_lim[34];   // (first[b] + count[b]), b <= 32
__shared__ unsigned long long sh_first[34];
__shared__ long long sh_off[35];

__device__ __noinline__ uint32_t slow_entry(const Tabs& t, uint32_t peek) {
    for (int b = kL1 + 1; b <= t.mx; b++) {
        const unsigned long long top = peek >> (32 - b);
        if (top < sh_lim[b]) {
            if (top < sh_first[b]) return kInvalid;
            return (t.symbols[sh_off[b] + (long long)(top - sh_first[b])] << 16) | (uint32_t)b;
        }
    }
    return kInvalid;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// table entry of the codeword at the top of `peek`
__device__ __forceinline__ uint32_t lookup(const Tabs& t, uint32_t peek) {
    uint32_t e = lds32(t.tab_s + ((peek >> (32 - kL1)) << 2));
    if ((e & 63u) == 0) {
        if (e & 0x40u) {
            const uint32_t k = (e >> 8) & 31u;
            e = lds32(t.tab_s + ((kL1Size + (e >> 16) + ((peek << kL1) >> (32 - k))) << 2));
        } else {
            e = slow_entry(t, peek);
        }
    }
    return e;
}

// Chunk bits staged in shared memory (big-endian words): a step is two LDS of
// the words under the bit position, a funnel shift and the table lookup.
// Positions are absolute bits of the staged window.
struct SmemReader {
    uint32_t base_s;   // shared address of word 0
    uint32_t a;        // bit position
    __device__ __forceinline__ void init(uint32_t bit) { a = bit; }
    __device__ __forceinline__ uint32_t pos() const { return a; }
    __device__ __forceinline__ uint32_t step(const Tabs& t) {
        const uint32_t wa = base_s + ((a >> 5) << 2);
        const uint32_t peek = __funnelshift_l(lds32(wa + 4), lds32(wa), a);
        const uint32_t e = lookup(t, peek);
        a += e & 63u;
        return e;
    }
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
    __device__ __forceinline__ void init(uint32_t bit) {
        const uint32_t i = bit >> 5;
        p = bit;
        s = bit & 31u;
        w0 = ld(i);
        w1 = ld(i + 1);
        wi = i + 2;
        w2 = ld(wi);
    }
    __device__ __forceinline__ uint32_t pos() const { return p; }
    __device__ __forceinline__ uint32_t step(const Tabs& t) {
        const uint32_t e = lookup(t, __funnelshift_l(w1, w0, s));
        const uint32_t len = e & 63u;
        const uint32_t s2 = s + len;
        p += len;
        if (s2 >= 32) {
            w0 = w1;
            w1 = w2;
            wi++;
            w2 = ld(wi);
        }
        s = s2 & 31u;
        return e;
    }
};

// Phase 1a: decode [A0, H) (H <= A0 + kWin) recording codeword starts
// relative to A0 in (lo, hi); counts into k, ORs entries into fl.
template <class Rd>
__device__ __forceinline__ void lane_head(const Tabs& t, Rd& rd, uint32_t A0, uint32_t H,
                                          uint32_t& k, uint32_t& fl, unsigned long long& lo,
                                          unsigned long long& hi) {
    const uint32_t h1 = A0 + 64 < H ? A0 + 64 : H;
    unsigned long long l = 0, h = 0;
    while (rd.pos() < h1) {
        l |= 1ull << (rd.pos() - A0);
        fl |= rd.step(t);
        k++;
    }
    while (rd.pos() < H) {
        h |= 1ull << (rd.pos() - A0 - 64);
        fl |= rd.step(t);
        k++;
    }
    lo = l;
    hi = h;
}

// Phase 1b: decode to the slice end S (exit = first codeword start >= S),
// then on into the next slice until a codeword start coincides with one of the
// next lane's head boundaries (nlo, nhi, relative to S) -- the synchronisation
// point -- or T is reached.  kt counts the codewords in [exit, sync).
template <class Rd>
__device__ __forceinline__ bool lane_rest(const Tabs& t, Rd& rd, uint32_t S, uint32_t T,
                                          unsigned long long nlo, unsigned long long nhi,
                                          uint32_t& k, uint32_t& fl, uint32_t& exit_pos,
                                          uint32_t& sync_pos, uint32_t& kt) {
    while (rd.pos() < S) {
        fl |= rd.step(t);
        k++;
    }
    exit_pos = rd.pos();
    uint32_t n = 0;
    bool found = false;
    while (rd.pos() < T) {
        const uint32_t r = rd.pos() - S;
        const unsigned long long m = r < 64 ? (nlo >> r) : (nhi >> (r - 64));
        if (m & 1ull) {
            found = true;
            break;
        }
        fl |= rd.step(t);
        n++;
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

// phase 3 of one lane: `count` codewords from `start`, must end at `end`
template <class Rd>
__device__ __forceinline__ bool lane_store(const Tabs& t, Rd& rd, uint32_t start, uint32_t end,
                                           uint32_t count, uint16_t* dst, uint32_t& zeros) {
    rd.init(start);
    uint32_t j = 0, z = 0, fl = 0;
    const uint32_t head = (uint32_t)umin((8u - (((uint32_t)(uintptr_t)dst >> 1) & 7u)) & 7u, count);
    for (; j < head; j++) {
        const uint32_t e = rd.step(t);
        fl |= e;
        dst[j] = (uint16_t)(e >> 16);
        z += e < 0x10000u;
    }
    for (; j + 8 <= count; j += 8) {
        uint32_t v[4];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const uint32_t e = rd.step(t);
            fl |= e;
            z += e < 0x10000u;
            if (q & 1) v[q >> 1] |= e & 0xFFFF0000u;
            else v[q >> 1] = e >> 16;
        }
        *reinterpret_cast<uint4*>(dst + j) = make_uint4(v[0], v[1], v[2], v[3]);
    }
    for (; j < count; j++) {
        const uint32_t e = rd.step(t);
        fl |= e;
        dst[j] = (uint16_t)(e >> 16);
        z += e < 0x10000u;
    }
    zeros += z;
    return !(fl & 0x80u) && rd.pos() == end;
}

// Phases 1-3 of one chunk by one warp; positions are absolute bits (the chunk
// occupies [sbit, sbit + B)).  false = hand the chunk back.
template <class Rd>
__device__ __forceinline__ bool decode_chunk(const Tabs& t, Rd rd, uint32_t sbit, uint32_t B,
                                             uint32_t cnt, uint16_t* out, uint32_t& zeros,
                                             DevStatus* st) {
    const uint32_t lane = lane_id();
    uint32_t L = B / kSliceMin;
    L = L < 1 ? 1 : (L > 32 ? 32 : L);
    const bool active = lane < L;
    const bool last = lane + 1 == L;
    const uint32_t s0 = sbit + (active ? (uint32_t)(((uint64_t)lane * B) / L) : B);
    const uint32_t s1 = sbit + (active ? (uint32_t)(((uint64_t)(lane + 1) * B) / L) : B);
    const uint32_t T = last || !active ? s1 : (s1 + kWin < sbit + B ? s1 + kWin : sbit + B);
    uint32_t k = 0, fl = 0, ex = s1, sp = s1, kt = 0, start = s0;
    unsigned long long lo = 0, hi = 0;
    bool fwd = false;   // this lane's tail met the next lane's path
    if (active) {
        rd.init(s0);
        lane_head(t, rd, s0, s0 + kWin < s1 ? s0 + kWin : s1, k, fl, lo, hi);
    }
    const unsigned long long nlo = __shfl_down_sync(kFull, lo, 1);
    const unsigned long long nhi = __shfl_down_sync(kFull, hi, 1);
    if (active) fwd = lane_rest(t, rd, s1, T, nlo, nhi, k, fl, ex, sp, kt);
    bool ok = !(fl & 0x80u);
    // phase 2: lane l is on the true path if lane l-1 is and l-1's tail met it;
    // the first lane that is not redecodes from its predecessor's exit
    bool restarted = lane == 0;
    uint32_t q = s0;   // start of the lane's true span
    for (uint32_t round = 0;; round++) {
        const bool pfwd = __shfl_up_sync(kFull, fwd, 1);
        const uint32_t pe = __shfl_up_sync(kFull, ex, 1);
        const uint32_t psp = __shfl_up_sync(kFull, sp, 1);
        const bool synced = !active || (ok && (restarted || pfwd));
        const unsigned bad = __ballot_sync(kFull, !synced);
        if (bad == 0) {
            if (active && !restarted) q = psp;
            break;
        }
        const uint32_t f = (uint32_t)(__ffs(bad) - 1);
        if (f == 0 || round >= L) return false;
        if (lane == f) {
            restarted = true;
            q = start = pe;
            k = 0;
            fl = 0;
            rd.init(pe);
            fwd = lane_rest(t, rd, s1, T, nlo, nhi, k, fl, ex, sp, kt);
            ok = !(fl & 0x80u);
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
    if (active && nl) ok3 = lane_store(t, rd, q, end, nl, out + o, z);
    if (!__all_sync(kFull, ok3)) return false;
    zeros += z;
    return true;
}

constexpr int kWarps = 8;

// dynamic shared memory: tables (kTabWords) then one staging buffer of
// `stage_words` words per warp
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
    uint32_t* stage = s_tab + kTabWords + wid * stage_words;
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
            good = decode_chunk(t, rd, sbit, B, cnt, out + base, zeros_total, st);
            __syncwarp();   // the stage is refilled by the next chunk
        } else {
            const uint64_t wbase = boff >> 2;
            GlobalReader rd;
            rd.w = words + wbase;
            rd.last = (uint32_t)umin(nwords > wbase ? nwords - 1 - wbase : 0, 0xFFFFFFFFull);
            good = decode_chunk(t, rd, (uint32_t)(boff & 3) * 8, B, cnt, out + base, zeros_total, st);
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
                         const uint32_t* symbols, int max_bw, uint32_t** tab_out) {
    int rc = SDQZ_OK;
    uint32_t* tab = scratch_as<uint32_t>(ctx, S_DTAB, kTabWords, &rc);
    if (!tab) return rc;
    dtab_kernel<<<1, 1024, 0, ctx->stream>>>(first, offsets, symbols, max_bw, ctx->d_status, tab);
    SDQZ_LAUNCHED_NAMED(ctx, "dtab_kernel");
    *tab_out = tab;
    return SDQZ_OK;
}

int launch_inflate_fast(sdqz_ctx* ctx, const uint8_t* payload, uint64_t nwords,
                        const uint32_t* chunk_bits, const unsigned long long* byte_off,
                        uint64_t n_chunks, uint32_t chunk, uint64_t n, const uint64_t* first,
                        const int64_t* offsets, const uint32_t* symbols, const uint32_t* tab,
                        int max_bw, uint16_t* codes, uint8_t* redo) {
    int rc = SDQZ_OK;
    unsigned int* counter = scratch_as<unsigned int>(ctx, S_COUNTER, 4, &rc);
    if (!counter) return rc;
    SDQZ_CUDA(ctx, cudaMemsetAsync(counter, 0, sizeof(unsigned int), ctx->stream));
    // per-warp staging: room for ~2x the average chunk (bigger chunks read global memory)
    const uint64_t avg = n_chunks ? (nwords * 4) / n_chunks : 0;
    uint32_t stage_words = 256;
    while (stage_words < 2048 && stage_words * 4 < 2 * avg + 64) stage_words <<= 1;
    const size_t smem = (kTabWords + (size_t)kWarps * stage_words) * 4;
    static size_t attr_smem = 0;
    if (smem > attr_smem) {
        cudaFuncSetAttribute(inflate_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_smem = smem;
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, inflate_fast_kernel, kWarps * 32, smem);
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = ceil_div(n_chunks, kWarps);
    const uint64_t cap = (uint64_t)ctx->num_sms * per_sm;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    inflate_fast_kernel<<<(unsigned)grid, kWarps * 32, smem, ctx->stream>>>(
        payload, nwords, chunk_bits, byte_off, n_chunks, chunk, n, first, offsets, symbols, tab,
        max_bw, codes, redo, counter, stage_words, ctx->d_status);
    SDQZ_LAUNCHED_NAMED(ctx, "inflate_fast_kernel");
    return SDQZ_OK;
}

}  // namespace sdqz
