// huffman.cu -- lossless stage on device (huffman.py):
//   K3  codebook: Huffman tree (two-queue merge over leaves sorted by
//       (freq, symbol), identical to the reference heap keyed on
//       (weight, min symbol), huffman.py:98-131) + canonical codebook
//       (huffman.py:146-190), one CTA;
//   K4  chunked encode + deflate (huffman.py:193-269): per-chunk bit counts,
//       one exclusive scan for byte offsets / outlier offsets, then a warp per
//       chunk packs codewords MSB-first (no atomics: each output word is
//       assembled by the lane that owns it) and compacts outliers in global
//       row-major order;
//   K5  inflate (huffman.py:272-356): a thread per chunk, 12-bit decode LUT in
//       shared memory, canonical fallback for longer codewords, the
//       reference's error checks in lockstep priority order.
#include "kernels.cuh"

namespace sdqz {

uint32_t default_chunk_size(uint64_t n) {   // huffman.py:206-212
    if (n == 0) return 256;
    double raw = (double)n / 2e4;
    uint64_t size = 1;
    if (raw > 1) {
        int e = (int)std::ceil(std::log2(raw));
        if (e < 0) e = 0;
        size = e >= 17 ? (1ull << 17) : (1ull << e);
    }
    if (size > 65536) size = 65536;
    if (size < 256) size = 256;
    return (uint32_t)size;
}

namespace {

// --------------------------------------------------------------------------
// histogram of uint32 codes (stage API; the fused path counts inside K2)
// --------------------------------------------------------------------------
__global__ void hist_u32_kernel(const uint32_t* __restrict__ codes, uint64_t n, uint32_t cap,
                                unsigned long long* hist, DevStatus* st) {
    extern __shared__ uint32_t sh[];
    bool use_smem = cap <= 16384;
    if (use_smem)
        for (uint32_t i = threadIdx.x; i < cap; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    bool bad = false;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c = codes[i];
        if (c >= cap) { bad = true; continue; }
        if (use_smem) atomicAdd(&sh[c], 1u);
        else atomicAdd(&hist[c], 1ull);
    }
    if (bad) atomicOr(&st->flags, (unsigned long long)F_CODE_RANGE);
    __syncthreads();
    if (use_smem)
        for (uint32_t i = threadIdx.x; i < cap; i += blockDim.x)
            if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
}

// --------------------------------------------------------------------------
// K3: codebook (single CTA)
// --------------------------------------------------------------------------
constexpr int kBookThreads = 1024;
constexpr uint32_t kSmemSortMax = 4096;

__device__ void bitonic_sort(unsigned long long* a, uint32_t m) {
    for (uint32_t k = 2; k <= m; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
                uint32_t ixj = i ^ j;
                if (ixj > i) {
                    unsigned long long x = a[i], y = a[ixj];
                    bool asc = (i & k) == 0;
                    if ((x > y) == asc) { a[i] = y; a[ixj] = x; }
                }
            }
            __syncthreads();
        }
    }
}

struct TreeScratch {       // global scratch for caps above the smem limit
    unsigned long long* keys;   // [cap]
    unsigned long long* iw;     // [cap]
    uint32_t* im;               // [cap]
    uint32_t* parent;           // [2*cap]
    uint32_t* dep;              // [2*cap] x2 (double buffer)
    uint32_t* jmp;              // [2*cap] x2
};

__global__ void __launch_bounds__(kBookThreads) codebook_kernel(
    const unsigned long long* __restrict__ hist, uint8_t* __restrict__ bw, uint32_t cap,
    BookDev book, DevStatus* st, int build_tree, int canon, TreeScratch gs) {
    extern __shared__ unsigned long long smem[];
    const bool small = cap <= kSmemSortMax;
    unsigned long long* keys = small ? smem : gs.keys;
    __shared__ uint32_t s_n, s_max, s_cnt[64], s_err;
    __shared__ unsigned long long s_first[64];
    __shared__ long long s_off[66];
    const uint32_t tid = threadIdx.x;

    if (build_tree) {
        // ---- leaves sorted by (freq, symbol) -------------------------------
        if (tid == 0) s_n = 0;
        __syncthreads();
        for (uint32_t s = tid; s < cap; s += blockDim.x) {
            unsigned long long f = hist[s];
            keys[s] = f ? ((f << 16) | s) : ~0ull;
            if (f) atomicAdd(&s_n, 1u);
        }
        __syncthreads();
        const uint32_t n = s_n;
        for (uint32_t s = tid; s < cap; s += blockDim.x) bw[s] = 0;
        if (n == 0) {
            if (tid == 0) atomicOr(&st->flags, (unsigned long long)F_ALL_ZERO_HIST);
            return;
        }
        bitonic_sort(keys, cap);
        if (n == 1) {
            if (tid == 0) bw[keys[0] & 0xFFFF] = 1;
            __syncthreads();
        } else {
            // ---- two-queue merge (thread 0) --------------------------------
            unsigned long long* iw = small ? (smem + cap) : gs.iw;
            uint32_t* im = small ? (uint32_t*)(smem + 2 * cap) : gs.im;
            uint32_t* parent = small ? (uint32_t*)(smem + 2 * cap) + cap : gs.parent;
            if (tid == 0) {
                uint32_t li = 0, ii = 0, ni = 0;
                unsigned long long lk = keys[0];
                for (uint32_t k = 0; k + 1 < n; k++) {
                    unsigned long long w[2];
                    uint32_t m[2], node[2];
#pragma unroll
                    for (int t = 0; t < 2; t++) {
                        bool take_leaf;
                        unsigned long long lw = lk >> 16;
                        uint32_t ls = (uint32_t)(lk & 0xFFFF);
                        if (ii == ni) take_leaf = true;
                        else if (li >= n) take_leaf = false;
                        else {
                            unsigned long long qw = iw[ii];
                            uint32_t qm = im[ii];
                            take_leaf = lw < qw || (lw == qw && ls < qm);
                        }
                        if (take_leaf) {
                            w[t] = lw; m[t] = ls; node[t] = li;
                            li++;
                            lk = li < n ? keys[li] : ~0ull;
                        } else {
                            w[t] = iw[ii]; m[t] = im[ii]; node[t] = n + ii;
                            ii++;
                        }
                    }
                    iw[ni] = w[0] + w[1];
                    im[ni] = min(m[0], m[1]);
                    ni++;
                    parent[node[0]] = n + k;
                    parent[node[1]] = n + k;
                }
            }
            __syncthreads();
            // ---- depths by pointer jumping (root = 2n-2) -------------------
            // d[v] = hops from v to jmp[v]; doubling: d += d[jmp], jmp = jmp[jmp].
            const uint32_t nodes = 2 * n - 1, root = 2 * n - 2;
            uint32_t* dc = small ? (uint32_t*)(smem + 2 * cap) + 3 * cap : gs.dep;
            uint32_t* jc = small ? dc + 2 * cap : gs.jmp;
            for (uint32_t v = tid; v < nodes; v += blockDim.x) {
                dc[v] = (v == root) ? 0 : 1;
                jc[v] = (v == root) ? root : parent[v];
            }
            __syncthreads();
            if (nodes <= 8 * blockDim.x) {
                // in place, staged through registers (<= 8 nodes per thread)
                for (int it = 0; it < 13; it++) {
                    uint32_t dv[8], jv[8];
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        uint32_t v = tid + q * blockDim.x;
                        if (v < nodes) {
                            uint32_t j = jc[v];
                            dv[q] = dc[v] + dc[j];
                            jv[q] = jc[j];
                        }
                    }
                    __syncthreads();
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        uint32_t v = tid + q * blockDim.x;
                        if (v < nodes) { dc[v] = dv[q]; jc[v] = jv[q]; }
                    }
                    __syncthreads();
                }
            } else {
                // ping-pong buffers in global scratch
                uint32_t *dn = gs.dep + 2 * cap, *jn = gs.jmp + 2 * cap;
                for (int it = 0; it < 18; it++) {
                    for (uint32_t v = tid; v < nodes; v += blockDim.x) {
                        uint32_t j = jc[v];
                        dn[v] = dc[v] + dc[j];
                        jn[v] = jc[j];
                    }
                    __syncthreads();
                    uint32_t* t = dc; dc = dn; dn = t;
                    t = jc; jc = jn; jn = t;
                }
            }
            for (uint32_t j = tid; j < n; j += blockDim.x) {
                uint32_t d = dc[j];
                bw[keys[j] & 0xFFFF] = (uint8_t)d;
            }
            __syncthreads();
        }
    }
    if (!canon) return;
    __syncthreads();

    // ---- canonical codebook from bitwidths (huffman.py:146-190) -------------
    if (tid < 64) { s_cnt[tid] = 0; }
    if (tid == 0) { s_n = 0; s_max = 0; s_err = 0; }
    __syncthreads();
    for (uint32_t s = tid; s < cap; s += blockDim.x) {
        uint32_t b = bw[s];
        book.entries[s] = 0;
        if (b) {
            atomicAdd(&s_n, 1u);
            atomicMax(&s_max, b);
            if (b < 64) atomicAdd(&s_cnt[b], 1u);
        }
    }
    __syncthreads();
    const uint32_t n = s_n, mx = s_max;
    if (tid == 0) {
        st->n_present = n;
        st->max_bw = mx;
        uint32_t err = 0;
        if (n == 0) err = F_NO_PRESENT;
        else if (mx > (uint32_t)kMaxBw) err = F_BW_TOO_BIG;
        else if (n >= 2) {
            unsigned long long kraft = 0;
            for (uint32_t b = 1; b <= mx; b++) kraft += (unsigned long long)s_cnt[b] << (mx - b);
            if (kraft != (1ull << mx)) err = F_KRAFT;
        }
        s_err = err;
        if (err) atomicOr(&st->flags, (unsigned long long)err);
        // first codes / offsets (huffman.py:170-176)
        unsigned long long code = 0;
        s_first[0] = 0;
        s_first[1] = 0;
        for (uint32_t b = 2; b <= 57; b++) {
            code = (code + (b - 1 <= mx ? s_cnt[b - 1] : 0)) << 1;
            s_first[b] = b <= mx ? code : 0;
        }
        long long run = 0;
        s_off[0] = 0;
        for (uint32_t b = 0; b <= 57; b++) {
            run += (b <= mx && b < 64) ? s_cnt[b] : 0;
            s_off[b + 1] = run;
        }
    }
    __syncthreads();
    if (s_err) return;
    const uint32_t unit = mx <= 24 ? 32 : 64;
    for (uint32_t b = tid; b < 58; b += blockDim.x) book.first[b] = s_first[b];
    for (uint32_t b = tid; b < 59; b += blockDim.x) book.offsets[b] = s_off[b];
    // order symbols by (bitwidth, symbol)
    for (uint32_t s = tid; s < cap; s += blockDim.x) {
        uint32_t b = bw[s];
        keys[s] = b ? (((unsigned long long)b << 16) | s) : ~0ull;
    }
    __syncthreads();
    bitonic_sort(keys, cap);
    for (uint32_t i = tid; i < n; i += blockDim.x) {
        unsigned long long k = keys[i];
        uint32_t s = (uint32_t)(k & 0xFFFF), b = (uint32_t)(k >> 16);
        unsigned long long cw = s_first[b] + (unsigned long long)(i - (uint32_t)s_off[b]);
        book.entries[s] = ((unsigned long long)b << (unit - 8)) | cw;
        book.symbols[i] = s;
    }
}

// decode LUT: entry = sym | len << 16; len 0 = longer than the LUT, 255 = no codeword
__global__ void lut_kernel(const uint64_t* __restrict__ first, const int64_t* __restrict__ offsets,
                           const uint32_t* __restrict__ symbols, int max_bw_arg,
                           const DevStatus* st, uint32_t* lut) {
    int mx = max_bw_arg > 0 ? max_bw_arg : (int)st->max_bw;
    if (mx < 1 || mx > kMaxBw) return;
    int lb = mx < kLutBits ? mx : kLutBits;
    long long nsym = offsets[mx + 1];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (1u << kLutBits);
         i += gridDim.x * blockDim.x) {
        uint32_t e = 0;
        if (i < (1u << lb)) {
            e = 0;
            bool found = false;
            for (int b = 1; b <= lb && !found; b++) {
                unsigned long long top = i >> (lb - b);
                unsigned long long cnt = (unsigned long long)(offsets[b + 1] - offsets[b]);
                if (top < first[b] + cnt) {
                    long long idx = offsets[b] + (long long)(top - first[b]);
                    if (idx < 0) idx = 0;
                    if (idx >= nsym) idx = nsym ? nsym - 1 : 0;
                    e = (symbols[idx] & 0xFFFF) | ((uint32_t)b << 16);
                    found = true;
                }
            }
            if (!found) e = (lb == mx) ? (255u << 16) : 0u;
        }
        lut[i] = e;
    }
}

// --------------------------------------------------------------------------
// K4: deflate
// --------------------------------------------------------------------------
enum Src { SRC_CODES = 0, SRC_U32 = 1, SRC_U64 = 2 };

template <int SRC>
__device__ __forceinline__ void fetch_unit(const void* src, const unsigned long long* table,
                                           uint64_t i, uint32_t cap, uint32_t unit, uint32_t& w,
                                           unsigned long long& cw, uint32_t& code, bool& bad) {
    unsigned long long u;
    if (SRC == SRC_CODES) {
        code = ((const uint16_t*)src)[i];
        if (code >= cap) { bad = true; w = 0; cw = 0; return; }
        if (!table) { w = 0; cw = 0; return; }   // outlier-only pass
        u = table[code];
    } else if (SRC == SRC_U32) {
        u = ((const uint32_t*)src)[i];
        code = 1;
    } else {
        u = ((const unsigned long long*)src)[i];
        code = 1;
    }
    w = (uint32_t)(u >> (unit - 8));
    cw = u & ((1ull << (unit - 8)) - 1);
}

struct DeflateArgs {
    const void* src;
    const unsigned long long* gtable;   // entries (codes source)
    uint64_t n;
    uint32_t chunk;
    uint64_t nchunks;
    uint32_t cap;
    uint32_t unit;                       // 32/64 (units source) or 0 => from status
    uint32_t* chunk_bits;
    uint32_t* chunk_zeros;
    unsigned long long* byte_off;
    unsigned long long* out_off;
    uint8_t* payload;
    unsigned long long payload_cap;
    const void* in;
    int in_kind;
    uint64_t in_split;
    const void* in_tail;
    uint64_t idx_base;
    unsigned long long* records;         // {idx, f64 bits} pairs
    unsigned long long out_cap;
    DevStatus* st;
};

__device__ __forceinline__ uint32_t unit_of(const DeflateArgs& a) {
    return a.unit ? a.unit : (a.st->max_bw <= 24 ? 32u : 64u);
}

// stats: warp per chunk -> bits, zero codes; flags range / absent-symbol errors
template <int SRC>
__global__ void __launch_bounds__(256) chunk_stats_kernel(DeflateArgs a) {
    extern __shared__ unsigned long long stable[];
    const uint32_t unit = unit_of(a);
    const bool smem_tab = SRC == SRC_CODES && a.cap <= 4096;
    if (smem_tab)
        for (uint32_t i = threadIdx.x; i < a.cap; i += blockDim.x) stable[i] = a.gtable[i];
    __syncthreads();
    const unsigned long long* tab = smem_tab ? stable : a.gtable;
    const uint32_t lane = lane_id();
    bool bad_range = false, bad_width = false;
    for (uint64_t c = blockIdx.x * 8ull + (threadIdx.x >> 5); c < a.nchunks; c += gridDim.x * 8ull) {
        uint64_t s = c * a.chunk, e = umin(s + a.chunk, a.n);
        uint32_t bits = 0, zeros = 0;
        for (uint64_t i = s + lane; i < e; i += 32) {
            uint32_t w, code;
            unsigned long long cw;
            fetch_unit<SRC>(a.src, tab, i, a.cap, unit, w, cw, code, bad_range);
            bits += w;
            zeros += (SRC == SRC_CODES && code == 0);
            if (w == 0 && (SRC != SRC_CODES || (tab && code < a.cap))) bad_width = true;
        }
        bits = __reduce_add_sync(kFull, bits);
        zeros = __reduce_add_sync(kFull, zeros);
        if (lane == 0) {
            a.chunk_bits[c] = bits;
            if (a.chunk_zeros) a.chunk_zeros[c] = zeros;
        }
    }
    unsigned long long f = 0;
    if (bad_range) f |= F_CODE_RANGE;
    if (bad_width) f |= (SRC == SRC_CODES) ? F_ABSENT_SYM : F_ZERO_WIDTH;
    if (f) atomicOr(&a.st->flags, f);
}

// exclusive scans over chunks (single CTA): byte offsets and outlier offsets
__global__ void __launch_bounds__(1024) chunk_scan_kernel(DeflateArgs a) {
    __shared__ unsigned long long sb[1024], so[1024];
    const uint64_t C = a.nchunks;
    const uint64_t per = ceil_div(C, blockDim.x);
    const uint64_t lo = umin(threadIdx.x * per, C), hi = umin(lo + per, C);
    unsigned long long tb = 0, to = 0;
    for (uint64_t c = lo; c < hi; c++) {
        tb += (a.chunk_bits[c] + 7) >> 3;
        if (a.chunk_zeros) to += a.chunk_zeros[c];
    }
    sb[threadIdx.x] = tb;
    so[threadIdx.x] = to;
    __syncthreads();
    for (uint32_t o = 1; o < blockDim.x; o <<= 1) {
        unsigned long long xb = threadIdx.x >= o ? sb[threadIdx.x - o] : 0;
        unsigned long long xo = threadIdx.x >= o ? so[threadIdx.x - o] : 0;
        __syncthreads();
        sb[threadIdx.x] += xb;
        so[threadIdx.x] += xo;
        __syncthreads();
    }
    unsigned long long rb = sb[threadIdx.x] - tb, ro = so[threadIdx.x] - to;
    for (uint64_t c = lo; c < hi; c++) {
        a.byte_off[c] = rb;
        if (a.out_off) a.out_off[c] = ro;
        rb += (a.chunk_bits[c] + 7) >> 3;
        if (a.chunk_zeros) ro += a.chunk_zeros[c];
    }
    if (threadIdx.x == blockDim.x - 1) {
        a.st->payload_bytes = sb[threadIdx.x];
        a.st->n_outliers = so[threadIdx.x];
        if (sb[threadIdx.x] > a.payload_cap || (a.records && so[threadIdx.x] > a.out_cap))
            atomicOr(&a.st->flags, (unsigned long long)F_OVERFLOW);
    }
}

__device__ __forceinline__ void store_word(uint8_t* payload, uint64_t wbyte, uint32_t word,
                                           uint64_t B, uint64_t Bend) {
    // word holds bytes [wbyte, wbyte+4) big-endian; write only [B, Bend)
    if (wbyte >= B && wbyte + 4 <= Bend) {
        *reinterpret_cast<uint32_t*>(payload + wbyte) = bswap32(word);
    } else {
        for (int k = 0; k < 4; k++) {
            uint64_t b = wbyte + k;
            if (b >= B && b < Bend) payload[b] = (uint8_t)(word >> (24 - 8 * k));
        }
    }
}

__device__ __forceinline__ double outlier_value(const DeflateArgs& a, uint64_t i, double two_eb) {
    const void* p = a.in;
    uint64_t j = i;
    if (i >= a.in_split) { p = a.in_tail; j = i - a.in_split; }
    double v = a.in_kind == 0 ? (double)((const float*)p)[j] : ((const double*)p)[j];
    return a.in_kind == 2 ? v : prequant(v, two_eb);
}

// pack: warp per chunk.  Lanes take 4 consecutive codes each and build a
// <=64-bit left-aligned segment; segments are concatenated by the owner-lane
// word assembly below (falls back to 1 code per lane when 4 codes overflow).
template <int SRC, bool PAYLOAD>
__global__ void __launch_bounds__(256) chunk_pack_kernel(DeflateArgs a) {
    extern __shared__ unsigned long long stable[];
    __shared__ unsigned long long s_seg[8][32];
    __shared__ uint32_t s_off[8][33];
    if (a.st->flags & (F_CODE_RANGE | F_ABSENT_SYM | F_ZERO_WIDTH | F_OVERFLOW | F_BW_TOO_BIG |
                       F_KRAFT | F_NO_PRESENT | F_ALL_ZERO_HIST))
        return;
    const uint32_t unit = unit_of(a);
    const bool smem_tab = SRC == SRC_CODES && a.cap <= 4096;
    if (smem_tab)
        for (uint32_t i = threadIdx.x; i < a.cap; i += blockDim.x) stable[i] = a.gtable[i];
    __syncthreads();
    const unsigned long long* tab = smem_tab ? stable : a.gtable;
    const double two_eb = a.st->two_eb;
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    unsigned long long* seg_s = s_seg[wid];
    uint32_t* off_s = s_off[wid];
    bool dummy = false;

    for (uint64_t c = blockIdx.x * 8ull + wid; c < a.nchunks; c += gridDim.x * 8ull) {
        const uint64_t s = c * a.chunk, e = umin(s + a.chunk, a.n);
        const uint64_t B = a.byte_off[c];
        const uint64_t Bend = B + ((a.chunk_bits[c] + 7) >> 3);
        uint64_t wbyte = B & ~3ull;                 // global byte of the current word 0
        uint32_t carry_bits = (uint32_t)(B & 3) * 8;
        uint32_t carry_word = 0;
        uint64_t orec = a.out_off ? a.out_off[c] : 0;

        auto emit = [&](unsigned long long seg, uint32_t len) {
            // concatenate the 32 lanes' segments onto the stream
            int total_l;
            uint32_t off = (uint32_t)warp_excl_scan((int)len, &total_l) + carry_bits;
            uint32_t total = carry_bits + (uint32_t)total_l;
            seg_s[lane] = seg;
            off_s[lane] = off;
            if (lane == 31) off_s[32] = total;
            __syncwarp();
            uint32_t nw = (total + 31) >> 5, full = total >> 5;
            uint32_t new_carry = 0;
            for (uint32_t j = lane; j < nw; j += 32) {
                uint32_t ws = 32 * j, we = ws + 32;
                uint32_t word = (j == 0) ? carry_word : 0;
                // first lane whose segment reaches past ws
                int lo = 0, hi = 31;
                while (lo < hi) {   // largest i with off[i] <= ws
                    int mid = (lo + hi + 1) >> 1;
                    if (off_s[mid] <= ws) lo = mid; else hi = mid - 1;
                }
                for (int i = lo; i < 32; i++) {
                    uint32_t o = off_s[i];
                    if (o >= we) break;
                    uint32_t oend = (i < 31) ? off_s[i + 1] : total;
                    if (oend <= ws) continue;
                    unsigned long long sg = seg_s[i];
                    uint32_t piece;
                    if (o >= ws) piece = (uint32_t)(sg >> 32) >> (o - ws);
                    else piece = (uint32_t)((sg << (ws - o)) >> 32);
                    word |= piece;
                }
                if (j < full) {
                    if (PAYLOAD) store_word(a.payload, wbyte + 4ull * j, word, B, Bend);
                } else {
                    new_carry = word;
                }
            }
            // broadcast the partial word from its owner
            uint32_t owner = (nw - 1) & 31;
            uint32_t pc = __shfl_sync(kFull, new_carry, owner);
            __syncwarp();
            if (total & 31) carry_word = pc; else carry_word = 0;
            wbyte += 4ull * full;
            carry_bits = total & 31;
        };

        for (uint64_t g = s; g < e; g += 128) {
            // lane owns codes g + 4*lane .. +3
            unsigned long long seg = 0;
            uint32_t len = 0, zc = 0;
            bool over = false;
            uint32_t codes4[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                uint64_t i = g + 4 * lane + k;
                codes4[k] = 1;
                if (i < e) {
                    uint32_t w, code;
                    unsigned long long cw;
                    fetch_unit<SRC>(a.src, tab, i, a.cap, unit, w, cw, code, dummy);
                    codes4[k] = code;
                    if (SRC == SRC_CODES && code == 0) zc++;
                    if (len + w <= 64) {
                        if (w) seg |= cw << (64 - len - w);
                    } else {
                        over = true;
                    }
                    len += w;
                }
            }
            if (PAYLOAD) {
                if (!__any_sync(kFull, over)) {
                    emit(seg, len);
                } else {
                    for (int k = 0; k < 4; k++) {
                        uint64_t i = g + 32 * k + lane;
                        unsigned long long sg = 0;
                        uint32_t w = 0;
                        if (i < e) {
                            uint32_t code;
                            unsigned long long cw;
                            fetch_unit<SRC>(a.src, tab, i, a.cap, unit, w, cw, code, dummy);
                            sg = w ? (cw << (64 - w)) : 0;
                        }
                        emit(sg, w);
                    }
                }
            }
            // outliers in row-major order
            if (SRC == SRC_CODES && a.records) {
                int ztot;
                uint32_t zoff = (uint32_t)warp_excl_scan((int)zc, &ztot);
                if (zc) {
                    uint64_t slot = orec + zoff;
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        uint64_t i = g + 4 * lane + k;
                        if (i < e && codes4[k] == 0) {
                            double v = outlier_value(a, i, two_eb);
                            a.records[2 * slot] = i + a.idx_base;
                            a.records[2 * slot + 1] = (unsigned long long)__double_as_longlong(v);
                            slot++;
                        }
                    }
                }
                orec += (uint64_t)ztot;
            }
        }
        // flush the final partial word
        if (PAYLOAD && carry_bits && lane == 0) store_word(a.payload, wbyte, carry_word, B, Bend);
        __syncwarp();
    }
}

// --------------------------------------------------------------------------
// encode (gather) for the stage API
// --------------------------------------------------------------------------
__global__ void encode_kernel(const uint32_t* __restrict__ codes, uint64_t n,
                              const unsigned long long* __restrict__ entries, uint32_t cap, int unit,
                              void* units, DevStatus* st) {
    bool bad_range = false, absent = false;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c = codes[i];
        unsigned long long u = 0;
        if (c >= cap) bad_range = true;
        else {
            u = entries[c];
            if (!u) absent = true;
        }
        if (unit == 32) ((uint32_t*)units)[i] = (uint32_t)u;
        else ((unsigned long long*)units)[i] = u;
    }
    unsigned long long f = (bad_range ? F_CODE_RANGE : 0) | (absent ? F_ABSENT_SYM : 0);
    if (f) atomicOr(&st->flags, f);
}

// --------------------------------------------------------------------------
// K5: inflate, thread per chunk
// --------------------------------------------------------------------------
__device__ __forceinline__ uint32_t load_be(const uint32_t* w, uint64_t i, uint64_t nw) {
    return i < nw ? bswap32(__ldg(w + i)) : 0u;   // zeros past the payload (huffman.py:338)
}

template <bool OUT32>
__global__ void __launch_bounds__(64) inflate_kernel(
    const uint8_t* __restrict__ payload, uint64_t nwords, const uint32_t* __restrict__ chunk_bits,
    const unsigned long long* __restrict__ byte_off, uint64_t nchunks, uint32_t chunk, uint64_t n,
    const uint64_t* __restrict__ gfirst, const int64_t* __restrict__ goffsets,
    const uint32_t* __restrict__ symbols, const uint32_t* __restrict__ glut, int max_bw_arg,
    void* out, DevStatus* st) {
    __shared__ uint32_t lut[1 << kLutBits];
    __shared__ unsigned long long first[58];
    __shared__ long long offs[59];
    for (uint32_t i = threadIdx.x; i < (1u << kLutBits); i += blockDim.x) lut[i] = glut[i];
    for (uint32_t i = threadIdx.x; i < 58; i += blockDim.x) first[i] = gfirst[i];
    for (uint32_t i = threadIdx.x; i < 59; i += blockDim.x) offs[i] = goffsets[i];
    __syncthreads();
    const int mx = max_bw_arg > 0 ? max_bw_arg : (int)st->max_bw;
    if (mx < 1 || mx > kMaxBw) return;
    const int lb = mx < kLutBits ? mx : kLutBits;
    const long long nsym = offs[mx + 1];
    const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t zeros = 0;
    if (c < nchunks) {
        const uint32_t* words = reinterpret_cast<const uint32_t*>(payload);
        const uint64_t sbit = byte_off[c] * 8;
        const uint32_t budget = chunk_bits[c];
        const uint64_t base = c * chunk;
        const uint64_t cnt = umin(chunk, n - base);
        uint64_t wi = sbit >> 5;
        uint32_t sh = (uint32_t)(sbit & 31);
        unsigned long long buf = (((unsigned long long)load_be(words, wi, nwords) << 32) |
                                  load_be(words, wi + 1, nwords)) << sh;
        int nb = 64 - (int)sh;
        wi += 2;
        uint32_t pos = 0;
        unsigned long long err = ~0ull;
        uint64_t k = 0;
        for (; k < cnt; k++) {
            if (nb <= 32) {
                buf |= (unsigned long long)load_be(words, wi, nwords) << (32 - nb);
                nb += 32;
                wi++;
            }
            uint32_t e = lut[buf >> (64 - lb)];
            uint32_t len = (e >> 16) & 0xFF;
            uint32_t sym = e & 0xFFFF;
            if (len == 0) {
                // canonical search beyond the LUT (huffman.py:295-305)
                uint64_t p = sbit + pos;
                uint64_t pw = p >> 5;
                uint32_t ps = (uint32_t)(p & 31);
                unsigned long long hi64 = ((unsigned long long)load_be(words, pw, nwords) << 32) | load_be(words, pw + 1, nwords);
                uint32_t w2 = load_be(words, pw + 2, nwords);
                unsigned long long peek64 = ps ? ((hi64 << ps) | (w2 >> (32 - ps))) : hi64;
                unsigned long long peek = peek64 >> (64 - mx);
                len = 255;
                for (int b = lb + 1; b <= mx; b++) {
                    unsigned long long top = peek >> (mx - b);
                    unsigned long long cntb = (unsigned long long)(offs[b + 1] - offs[b]);
                    if (top < first[b] + cntb) {
                        long long idx = offs[b] + (long long)(top - first[b]);
                        if (idx < 0) idx = 0;
                        if (idx >= nsym) idx = nsym ? nsym - 1 : 0;
                        sym = symbols[idx];
                        len = b;
                        break;
                    }
                }
            }
            if (len == 255) { err = k * 4 + DK_NO_CODEWORD; break; }
            if (pos + len > budget) { err = k * 4 + DK_EXHAUSTED; break; }
            if (OUT32) ((uint32_t*)out)[base + k] = sym;
            else ((uint16_t*)out)[base + k] = (uint16_t)sym;
            zeros += (sym == 0);
            pos += len;
            if (len < 64) buf <<= len; else buf = 0;
            nb -= (int)len;
            if (nb < 0) {   // only after a long codeword: resync the window from memory
                uint64_t p = sbit + pos;
                wi = p >> 5;
                sh = (uint32_t)(p & 31);
                buf = (((unsigned long long)load_be(words, wi, nwords) << 32) | load_be(words, wi + 1, nwords)) << sh;
                nb = 64 - (int)sh;
                wi += 2;
            }
        }
        if (err == ~0ull && pos != budget) err = (0x3fffffffffffffffull << 2) | DK_DISAGREE;
        if (err != ~0ull) atomicMin(&st->decode_key, err);
    }
    zeros = __reduce_add_sync(kFull, zeros);
    if (lane_id() == 0 && zeros) atomicAdd(&st->n_zero, (unsigned long long)zeros);
}

template <int SRC>
int run_deflate(sdqz_ctx* ctx, DeflateArgs& a, bool payload) {
    size_t smem = (SRC == SRC_CODES && a.cap <= 4096) ? a.cap * 8 : 0;
    uint64_t grid = ceil_div(a.nchunks, 8);
    if (grid > (uint64_t)ctx->num_sms * 16) grid = ctx->num_sms * 16;
    if (grid < 1) grid = 1;
    chunk_stats_kernel<SRC><<<(unsigned)grid, 256, smem, ctx->stream>>>(a);
    SDQZ_LAUNCHED(ctx);
    chunk_scan_kernel<<<1, 1024, 0, ctx->stream>>>(a);
    SDQZ_LAUNCHED(ctx);
    if (payload)
        chunk_pack_kernel<SRC, true><<<(unsigned)grid, 256, smem, ctx->stream>>>(a);
    else
        chunk_pack_kernel<SRC, false><<<(unsigned)grid, 256, smem, ctx->stream>>>(a);
    SDQZ_LAUNCHED(ctx);
    return SDQZ_OK;
}

}  // namespace

int launch_histogram_u32(sdqz_ctx* ctx, const uint32_t* codes, uint64_t n, uint32_t cap,
                         unsigned long long* hist) {
    size_t smem = cap <= 16384 ? cap * 4 : 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(hist_u32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    uint64_t grid = ceil_div(n, 256);
    if (grid > (uint64_t)ctx->num_sms * 4) grid = ctx->num_sms * 4;
    if (grid < 1) grid = 1;
    hist_u32_kernel<<<(unsigned)grid, 256, smem, ctx->stream>>>(codes, n, cap, hist, ctx->d_status);
    SDQZ_LAUNCHED(ctx);
    return SDQZ_OK;
}

int launch_codebook(sdqz_ctx* ctx, const unsigned long long* d_hist, uint8_t* d_bw, uint32_t cap,
                    const BookDev& book, bool build_tree, bool canon, bool err_format) {
    (void)err_format;
    int rc = SDQZ_OK;
    TreeScratch gs{};
    size_t smem = 0;
    if (cap <= kSmemSortMax) {
        // keys (cap u64) + iw (cap u64) + im/parent/dep/jmp (u32: cap + 2cap + 2cap + 2cap)
        smem = cap * 8 * 2 + cap * 4 * 7;
    } else {
        unsigned long long* base = scratch_as<unsigned long long>(ctx, S_TREE, (size_t)cap * 12, &rc);
        if (!base) return rc;
        gs.keys = base;
        gs.iw = base + cap;
        uint32_t* u = (uint32_t*)(base + 2 * cap);
        gs.im = u;
        gs.parent = u + cap;
        gs.dep = u + 3 * cap;
        gs.jmp = u + 7 * cap;
    }
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(codebook_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    codebook_kernel<<<1, kBookThreads, smem, ctx->stream>>>(d_hist, d_bw, cap, book, ctx->d_status,
                                                           build_tree ? 1 : 0, canon ? 1 : 0, gs);
    SDQZ_LAUNCHED(ctx);
    return SDQZ_OK;
}

int launch_build_lut(sdqz_ctx* ctx, const uint64_t* first, const int64_t* offsets,
                     const uint32_t* symbols, int max_bw_or_neg, uint32_t* lut) {
    lut_kernel<<<16, 256, 0, ctx->stream>>>(first, offsets, symbols, max_bw_or_neg, ctx->d_status, lut);
    SDQZ_LAUNCHED(ctx);
    return SDQZ_OK;
}

int launch_deflate(sdqz_ctx* ctx, const DeflateJob& job) {
    int rc = SDQZ_OK;
    DeflateArgs a{};
    a.n = job.n;
    a.chunk = job.chunk;
    a.nchunks = ceil_div(job.n, job.chunk);
    a.cap = job.cap;
    a.gtable = (const unsigned long long*)job.entries;
    a.chunk_bits = job.chunk_bits;
    a.payload = job.payload;
    a.payload_cap = job.payload_cap;
    a.in = job.in;
    a.in_kind = job.in_kind;
    a.in_split = job.in_split;
    a.in_tail = job.in_tail;
    a.idx_base = job.idx_base;
    a.records = (unsigned long long*)job.out_records;
    a.out_cap = job.out_cap;
    a.st = ctx->d_status;
    if (a.nchunks == 0) return SDQZ_OK;
    a.byte_off = scratch_as<unsigned long long>(ctx, S_BYTE_OFF, a.nchunks, &rc);
    if (!a.byte_off) return rc;
    if (job.codes) {
        a.src = job.codes;
        a.unit = 0;
        a.chunk_zeros = scratch_as<uint32_t>(ctx, S_CHUNK_AUX, a.nchunks, &rc);
        a.out_off = scratch_as<unsigned long long>(ctx, S_OUT_OFF, a.nchunks, &rc);
        if (!a.chunk_zeros || !a.out_off) return rc;
        return run_deflate<SRC_CODES>(ctx, a, job.want_payload);
    }
    a.src = job.units;
    a.unit = job.units_width;
    a.chunk_zeros = nullptr;
    a.out_off = nullptr;
    a.records = nullptr;
    if (job.units_width == 32) return run_deflate<SRC_U32>(ctx, a, true);
    return run_deflate<SRC_U64>(ctx, a, true);
}

int launch_encode_u32(sdqz_ctx* ctx, const uint32_t* codes, uint64_t n, const uint64_t* entries,
                      uint32_t cap, int unit, void* units) {
    uint64_t grid = ceil_div(n, 256);
    if (grid > (uint64_t)ctx->num_sms * 8) grid = ctx->num_sms * 8;
    if (grid < 1) grid = 1;
    encode_kernel<<<(unsigned)grid, 256, 0, ctx->stream>>>(codes, n, (const unsigned long long*)entries,
                                                          cap, unit, units, ctx->d_status);
    SDQZ_LAUNCHED(ctx);
    return SDQZ_OK;
}

int launch_inflate(sdqz_ctx* ctx, const uint8_t* payload, uint64_t payload_bytes,
                   const uint32_t* chunk_bits, uint64_t n_chunks, uint32_t chunk,
                   const uint64_t* first, const int64_t* offsets, const uint32_t* symbols,
                   const uint32_t* lut, int max_bw, uint64_t n, void* codes, bool out32) {
    // readable words: the payload plus its zero padding (callers pad >= 16 bytes)
    const uint64_t nwords = (payload_bytes + 16) / 4;
    int rc = SDQZ_OK;
    if (n_chunks == 0) return SDQZ_OK;
    // byte offsets of chunks (scan of ceil(bits/8)); the scan also totals the payload
    DeflateArgs a{};
    a.nchunks = n_chunks;
    a.chunk_bits = const_cast<uint32_t*>(chunk_bits);
    a.chunk_zeros = nullptr;
    a.out_off = nullptr;
    a.records = nullptr;
    a.payload_cap = ~0ull;
    a.st = ctx->d_status;
    a.byte_off = scratch_as<unsigned long long>(ctx, S_BYTE_OFF, n_chunks, &rc);
    if (!a.byte_off) return rc;
    chunk_scan_kernel<<<1, 1024, 0, ctx->stream>>>(a);
    SDQZ_LAUNCHED(ctx);
    uint64_t grid = ceil_div(n_chunks, 64);
    if (out32)
        inflate_kernel<true><<<(unsigned)grid, 64, 0, ctx->stream>>>(
            payload, nwords, chunk_bits, a.byte_off, n_chunks, chunk, n, first, offsets, symbols, lut,
            max_bw, codes, ctx->d_status);
    else
        inflate_kernel<false><<<(unsigned)grid, 64, 0, ctx->stream>>>(
            payload, nwords, chunk_bits, a.byte_off, n_chunks, chunk, n, first, offsets, symbols, lut,
            max_bw, codes, ctx->d_status);
    SDQZ_LAUNCHED(ctx);
    return SDQZ_OK;
}

}  // namespace sdqz
