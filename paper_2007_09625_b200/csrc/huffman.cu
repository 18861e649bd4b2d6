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
#include "scan.cuh"

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

// Bitonic sort of 1024 u64 keys held one per thread (blockDim == 1024):
// strides < 32 exchange through shuffles, larger ones through `a` (smem).
__device__ unsigned long long bitonic_sort_1024(unsigned long long x, unsigned long long* a) {
    const uint32_t i = threadIdx.x;
    for (uint32_t k = 2; k <= 1024; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            unsigned long long y;
            if (j >= 32) {
                a[i] = x;
                __syncthreads();
                y = a[i ^ j];
                __syncthreads();
            } else {
                y = __shfl_xor_sync(kFull, x, j);
            }
            const bool asc = (i & k) == 0, low = (i & j) == 0;
            const unsigned long long mn = x < y ? x : y, mxv = x < y ? y : x;
            x = (low == asc) ? mn : mxv;
        }
    }
    return x;
}

struct TreeScratch {       // global scratch for caps above the smem limit
    unsigned long long* keys;   // [cap]
    unsigned long long* iw;     // [cap]
    uint32_t* im;               // [cap]
    uint32_t* parent;           // [2*cap]
    uint32_t* dep;              // [2*cap] x2 (double buffer)
    uint32_t* jmp;              // [2*cap] x2
};

#ifdef SDQZ_DEBUG_TIMING
#define BOOK_T(i) do { __syncthreads(); if (threadIdx.x == 0) tclk[i] = clock64(); } while (0)
#else
#define BOOK_T(i) do {} while (0)
#endif

template <bool SMALL>
__global__ void __launch_bounds__(kBookThreads) codebook_kernel(
    const unsigned long long* __restrict__ hist, uint8_t* __restrict__ bw, uint32_t cap,
    BookDev book, DevStatus* st, int build_tree, int canon, TreeScratch gs, uint32_t round_min) {
    extern __shared__ unsigned long long smem[];
    // SMALL (cap <= 4096): every table lives in shared memory; the template
    // keeps the pointers in the shared address space (no generic accesses)
    constexpr bool small = SMALL;
    unsigned long long* keys = small ? smem : gs.keys;
    __shared__ uint32_t s_n, s_max, s_cnt[64], s_err;
    __shared__ unsigned long long s_first[64];
    __shared__ long long s_off[66];
    const uint32_t tid = threadIdx.x;
#ifdef SDQZ_DEBUG_TIMING
    __shared__ long long tclk[8];
    if (tid < 8) tclk[tid] = 0;
#endif
    BOOK_T(0);

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
        BOOK_T(1);
        if (cap <= 1024 && blockDim.x == 1024) {
            __shared__ unsigned long long xbuf[1024];
            const unsigned long long x = bitonic_sort_1024(tid < cap ? keys[tid] : ~0ull, xbuf);
            __syncthreads();
            if (tid < cap) keys[tid] = x;
            __syncthreads();
        } else {
            bitonic_sort(keys, cap);
        }
        BOOK_T(2);
        if (n == 1) {
            if (tid == 0) bw[keys[0] & 0xFFFF] = 1;
            __syncthreads();
        } else {
            // ---- two-queue merge (thread 0) --------------------------------
            // Internal nodes are keyed like leaves, (weight << 16) | min symbol,
            // so one u64 compare orders both queues exactly as the reference
            // heap does.  Three-deep register windows over each queue keep the
            // shared-memory loads off the sequential critical path.
            unsigned long long* iq = small ? (smem + cap) : gs.iw;
            uint32_t* parent = small ? (uint32_t*)(smem + 2 * cap) + cap : gs.parent;
            constexpr unsigned long long NONE = ~0ull;
            // -- parallel rounds.  With t = the first node the sequential merge
            // would create (sum of the two smallest frontier keys), every
            // frontier element below t is popped before t, pairwise in sorted
            // order; so the first 2*floor(m/2) of the m elements below t can be
            // merged in one round, exactly as the heap would.  Rounds continue
            // while they stay productive; the tail runs sequentially.
            // The frontier state (li, ii, ni) is block-uniform and kept in every
            // thread's registers; t and the counts below t are computed by all
            // threads (broadcast reads + barrier counts), so a round has no
            // serial section.
            unsigned long long* fk = small ? (unsigned long long*)((uint32_t*)(smem + 2 * cap) + 3 * cap)
                                           : (unsigned long long*)gs.dep;
            uint32_t* fid = small ? (uint32_t*)(smem + 2 * cap) + 5 * cap : gs.jmp;
            auto lower = [](const unsigned long long* a, uint32_t lo, uint32_t hi,
                            unsigned long long key) {
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (a[mid] < key) lo = mid + 1; else hi = mid;
                }
                return lo;
            };
            uint32_t li = 0, ii = 0, ni = 0;
            __shared__ uint32_t r_li, r_ii, r_ni;
            while (ni + 1 < n) {
                const unsigned long long LH = li < n ? keys[li] : NONE, IH = ii < ni ? iq[ii] : NONE;
                unsigned long long f0, f1;
                if (LH < IH) {
                    f0 = LH;
                    const unsigned long long L1 = li + 1 < n ? keys[li + 1] : NONE;
                    f1 = L1 < IH ? L1 : IH;
                } else {
                    f0 = IH;
                    const unsigned long long I1 = ii + 1 < ni ? iq[ii + 1] : NONE;
                    f1 = LH < I1 ? LH : I1;
                }
                const unsigned long long t =
                    (((f0 >> 16) + (f1 >> 16)) << 16) | min(f0 & 0xFFFF, f1 & 0xFFFF);
                // elements below t in each (sorted) queue
                uint32_t mL = 0, mI = 0;
                for (uint32_t j0 = 0; j0 < n - li; j0 += blockDim.x) {
                    const uint32_t j = li + j0 + tid;
                    mL += __syncthreads_count(j < n && keys[j] < t);
                }
                for (uint32_t j0 = 0; j0 < ni - ii; j0 += blockDim.x) {
                    const uint32_t j = ii + j0 + tid;
                    mI += __syncthreads_count(j < ni && iq[j] < t);
                }
                const uint32_t p = (mL + mI) / 2;
                if (p < round_min) break;   // unproductive: finish sequentially
                // merged position of every element below t
                for (uint32_t j = tid; j < mL + mI; j += blockDim.x) {
                    unsigned long long key;
                    uint32_t pos, id;
                    if (j < mL) {
                        key = keys[li + j];
                        pos = j + (lower(iq, ii, ii + mI, key) - ii);
                        id = li + j;
                    } else {
                        const uint32_t q = j - mL;
                        key = iq[ii + q];
                        pos = q + (lower(keys, li, li + mL, key) - li);
                        id = n + ii + q;
                    }
                    if (pos < 2 * p) { fk[pos] = key; fid[pos] = id; }
                }
                uint32_t cL = mL, cI = mI;
                if ((mL + mI) & 1) {   // the largest element below t waits for the next round
                    const bool last_leaf = mL > 0 && (mI == 0 || keys[li + mL - 1] > iq[ii + mI - 1]);
                    if (last_leaf) cL--; else cI--;
                }
                __syncthreads();
                for (uint32_t j = tid; j < p; j += blockDim.x) {
                    const unsigned long long a = fk[2 * j], b = fk[2 * j + 1];
                    iq[ni + j] = (((a >> 16) + (b >> 16)) << 16) | min(a & 0xFFFF, b & 0xFFFF);
                    parent[fid[2 * j]] = n + ni + j;
                    parent[fid[2 * j + 1]] = n + ni + j;
                }
                li += cL;
                ii += cI;
                ni += p;
                __syncthreads();
            }
            if (tid == 0) { r_li = li; r_ii = ii; r_ni = ni; }
            __syncthreads();
            BOOK_T(3);
            // -- sequential tail (thread 0): two-queue merge from (li, ii, ni)
            if (tid == 0) {
                uint32_t li = r_li, ii = r_ii, ni = r_ni;
                auto lk = [&](uint32_t i) { return i < n ? keys[i] : NONE; };
                auto ik = [&](uint32_t i) { return i < ni ? iq[i] : NONE; };
                unsigned long long L0 = lk(li), L1 = lk(li + 1), L2 = lk(li + 2);
                unsigned long long H0 = ik(ii), H1 = ik(ii + 1), H2 = ik(ii + 2);
                for (uint32_t k = ni; k + 1 < n; k++) {
                    unsigned long long kk[2];
                    uint32_t node[2];
#pragma unroll
                    for (int t = 0; t < 2; t++) {
                        // branch-free pick; both candidate refills are loaded
                        // every step
                        const bool leaf = L0 < H0;
                        const unsigned long long ln = (li + 3 < n) ? keys[li + 3] : NONE;
                        const unsigned long long hn = (ii + 3 < ni) ? iq[ii + 3] : NONE;
                        kk[t] = leaf ? L0 : H0;
                        node[t] = leaf ? li : n + ii;
                        L0 = leaf ? L1 : L0;
                        L1 = leaf ? L2 : L1;
                        L2 = leaf ? ln : L2;
                        H0 = leaf ? H0 : H1;
                        H1 = leaf ? H1 : H2;
                        H2 = leaf ? H2 : hn;
                        li += leaf;
                        ii += !leaf;
                    }
                    const unsigned long long nk =
                        (((kk[0] >> 16) + (kk[1] >> 16)) << 16) | min(kk[0] & 0xFFFF, kk[1] & 0xFFFF);
                    iq[ni] = nk;
                    const uint32_t d = ni - ii;
                    if (d == 0) H0 = nk;
                    else if (d == 1) H1 = nk;
                    else if (d == 2) H2 = nk;
                    ni++;
                    parent[node[0]] = n + k;
                    parent[node[1]] = n + k;
                }
                (void)ni;
            }
            __syncthreads();
            BOOK_T(4);
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
                // in place, staged through registers (<= 8 nodes per thread);
                // stops once every node points at the root (~log2 of the depth)
                for (int it = 0; it < 13; it++) {
                    uint32_t dv[8], jv[8];
                    bool done = true;
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        uint32_t v = tid + q * blockDim.x;
                        if (v < nodes) {
                            uint32_t j = jc[v];
                            dv[q] = dc[v] + dc[j];
                            jv[q] = jc[j];
                            done &= j == root;
                        }
                    }
                    if (__syncthreads_and(done)) break;
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
    BOOK_T(5);
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
    // order symbols by (bitwidth, symbol) without sorting: a symbol's rank in
    // its bitwidth group = same-width symbols before it (match_any within the
    // warp + per-(warp, width) counts scanned down the warps), tile by tile
    __shared__ uint32_t wcnt[32][64];
    __shared__ uint32_t run[64];
    if (tid < 64) run[tid] = 0;
    const uint32_t lane = tid & 31, wid = tid >> 5;
    BOOK_T(6);
    for (uint32_t base = 0; base < cap; base += blockDim.x) {
        const uint32_t s = base + tid;
        const uint32_t b = s < cap ? bw[s] : 0;
        const uint32_t m = __match_any_sync(kFull, b);
        const uint32_t rk = __popc(m & ((1u << lane) - 1));
        for (uint32_t i = tid; i < 32 * 64; i += blockDim.x) (&wcnt[0][0])[i] = 0;
        __syncthreads();
        if (rk == 0 && b < 64) wcnt[wid][b] = __popc(m);
        __syncthreads();
        if (tid < 64) {
            uint32_t acc = run[tid];
            for (uint32_t w = 0; w < blockDim.x / 32; w++) {
                const uint32_t v = wcnt[w][tid];
                wcnt[w][tid] = acc;
                acc += v;
            }
            run[tid] = acc;
        }
        __syncthreads();
        if (b && b < 64) {
            const uint32_t i = (uint32_t)s_off[b] + wcnt[wid][b] + rk;
            book.entries[s] = ((unsigned long long)b << (unit - 8)) |
                              (s_first[b] + (unsigned long long)(i - (uint32_t)s_off[b]));
            book.symbols[i] = s;
        }
        __syncthreads();
    }
    BOOK_T(7);
#ifdef SDQZ_DEBUG_TIMING
    if (tid == 0) printf("codebook phases(cycles): keys %lld sort %lld merge-rounds %lld tail %lld depths %lld canon-prep %lld canon-rank %lld\n",
                         tclk[1]-tclk[0], tclk[2]-tclk[1], tclk[3]-tclk[2], tclk[4]-tclk[3], tclk[5]-tclk[4], tclk[6]-tclk[5], tclk[7]-tclk[6]);
#endif
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
            if (!found && lb == mx) {
                e = 255u << 16;
            } else if (!found) {
                // longer than the LUT: record the shortest width any codeword
                // with this prefix can have, so the decoder's canonical search
                // starts there (len field 0, hint in the symbol field)
                const unsigned long long pmin = (unsigned long long)i << (mx - lb);
                uint32_t b0 = (uint32_t)mx + 1;
                for (int b = lb + 1; b <= mx; b++) {
                    const unsigned long long cnt = (unsigned long long)(offsets[b + 1] - offsets[b]);
                    if (pmin < ((first[b] + cnt) << (mx - b))) { b0 = (uint32_t)b; break; }
                }
                e = b0;
            }
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
    uint64_t rec_limit;                  // records only for indices below (sharded: own slab)
    unsigned long long* records;         // {idx, f64 bits} pairs
    unsigned long long out_cap;
    const double* heads;                 // block-head outlier values (i % 32 == 0, i < heads_limit)
    uint64_t heads_limit;
    DevStatus* st;
    bool trusted;
};

__device__ __forceinline__ uint32_t unit_of(const DeflateArgs& a) {
    return a.unit ? a.unit : (a.st->max_bw <= 24 ? 32u : 64u);
}

// Eight consecutive codes per lane: one 16-byte load when the group is
// aligned and complete, scalar loads otherwise.
template <int SRC>
__device__ __forceinline__ void load_group8(const DeflateArgs& a, uint64_t i0, uint64_t e,
                                            uint32_t codes[8], bool& valid_all) {
    if (SRC == SRC_CODES && (i0 & 7) == 0 && i0 + 8 <= e) {
        uint4 v = __ldg(reinterpret_cast<const uint4*>((const uint16_t*)a.src + i0));
        codes[0] = v.x & 0xFFFF; codes[1] = v.x >> 16;
        codes[2] = v.y & 0xFFFF; codes[3] = v.y >> 16;
        codes[4] = v.z & 0xFFFF; codes[5] = v.z >> 16;
        codes[6] = v.w & 0xFFFF; codes[7] = v.w >> 16;
        valid_all = true;
        return;
    }
    valid_all = false;
#pragma unroll
    for (int k = 0; k < 8; k++) codes[k] = 0;
}

template <int SRC>
__device__ __forceinline__ void unit_of_code(const DeflateArgs& a, const unsigned long long* tab,
                                             uint64_t i, uint32_t code, bool have_code,
                                             uint32_t unit, uint32_t& w, unsigned long long& cw,
                                             uint32_t& c_out, bool& bad_range) {
    if (SRC == SRC_CODES && have_code) {
        c_out = code;
        if (code >= a.cap) { bad_range = true; w = 0; cw = 0; return; }
        if (!tab) { w = 0; cw = 0; return; }
        unsigned long long u = tab[code];
        w = (uint32_t)(u >> (unit - 8));
        cw = u & ((1ull << (unit - 8)) - 1);
        return;
    }
    fetch_unit<SRC>(a.src, tab, i, a.cap, unit, w, cw, c_out, bad_range);
}

__device__ __forceinline__ bool zero_half16(uint32_t w) {   // either 16-bit half == 0
    return ((w - 0x00010001u) & ~w & 0x80008000u) != 0;
}

// stats for codes produced by K2 (always < cap, every symbol present in the
// book): a byte table of widths, two lookups per 32-bit word, zero codes
// counted exactly only in words that hold one (rare)
__global__ void __launch_bounds__(256) chunk_stats_fast_kernel(DeflateArgs a) {
    __shared__ uint8_t s_w[4096];
    const uint32_t wshift = unit_of(a) - 8;
    for (uint32_t i = threadIdx.x; i < a.cap; i += blockDim.x) s_w[i] = (uint8_t)(a.gtable[i] >> wshift);
    __syncthreads();
    const uint32_t lane = lane_id();
    const uint16_t* src = (const uint16_t*)a.src;
    for (uint64_t c = blockIdx.x * 8ull + (threadIdx.x >> 5); c < a.nchunks; c += gridDim.x * 8ull) {
        const uint64_t s = c * a.chunk, e = umin(s + a.chunk, a.n);
        uint32_t bits = 0, zeros = 0;
        uint64_t i0 = s + 8 * lane;
        if ((s & 7) == 0) {
            auto acc4 = [&](const uint4& v) {
                const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    bits += (uint32_t)s_w[wv[k] & 0xFFFF] + (uint32_t)s_w[wv[k] >> 16];
                    if (zero_half16(wv[k])) zeros += ((wv[k] & 0xFFFF) == 0) + ((wv[k] >> 16) == 0);
                }
            };
            // four 16-byte loads per lane in flight (a chunk is a few such rounds)
            for (; i0 + 3 * 256 + 8 <= e; i0 += 4 * 256) {
                uint4 v[4];
#pragma unroll
                for (int u = 0; u < 4; u++) v[u] = __ldg(reinterpret_cast<const uint4*>(src + i0 + u * 256));
#pragma unroll
                for (int u = 0; u < 4; u++) acc4(v[u]);
            }
            for (; i0 + 8 <= e; i0 += 256) acc4(__ldg(reinterpret_cast<const uint4*>(src + i0)));
        }
        for (; i0 < e; i0 += 256) {   // unaligned chunk or ragged tail
#pragma unroll
            for (int k = 0; k < 8; k++) {
                if (i0 + k < e) {
                    const uint32_t code = src[i0 + k];
                    bits += s_w[code];
                    zeros += code == 0;
                }
            }
        }
        bits = __reduce_add_sync(kFull, bits);
        zeros = __reduce_add_sync(kFull, zeros);
        if (lane == 0) {
            a.chunk_bits[c] = bits;
            if (a.chunk_zeros) a.chunk_zeros[c] = zeros;
        }
    }
}

// stats: warp per chunk -> bits, zero codes; flags range / absent-symbol errors
// TS: the codebook (cap <= 4096) is staged in shared memory; as a template
// parameter it keeps table reads in the shared address space.
template <int SRC, bool TS>
__global__ void __launch_bounds__(256) chunk_stats_kernel(DeflateArgs a) {
    extern __shared__ unsigned long long stable[];
    const uint32_t unit = unit_of(a);
    if (TS)
        for (uint32_t i = threadIdx.x; i < a.cap; i += blockDim.x) stable[i] = a.gtable[i];
    __syncthreads();
    const unsigned long long* tab = TS ? stable : a.gtable;
    const uint32_t lane = lane_id();
    bool bad_range = false, bad_width = false;
    for (uint64_t c = blockIdx.x * 8ull + (threadIdx.x >> 5); c < a.nchunks; c += gridDim.x * 8ull) {
        const uint64_t s = c * a.chunk, e = umin(s + a.chunk, a.n);
        uint32_t bits = 0, zeros = 0;
        if (SRC == SRC_CODES && ((s | e) & 7) == 0) {
            // aligned chunk: 16-byte loads of 8 codes, branch-free accumulation
            const uint16_t* src = (const uint16_t*)a.src;
            const uint32_t wshift = unit - 8;
            for (uint64_t i0 = s + 8 * lane; i0 < e; i0 += 256) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + i0));
                const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const uint32_t code = (wv[k >> 1] >> (16 * (k & 1))) & 0xFFFF;
                    const bool inr = code < a.cap;
                    const unsigned long long u = (inr && tab) ? tab[code] : 0ull;
                    bad_range |= !inr;
                    bad_width |= tab && inr && u == 0;
                    bits += (uint32_t)(u >> wshift);
                    zeros += code == 0;
                }
            }
        } else
        for (uint64_t g = s; g < e; g += 256) {
            const uint64_t i0 = g + 8 * lane;
            uint32_t codes[8];
            bool vec;
            load_group8<SRC>(a, i0, e, codes, vec);
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const uint64_t i = i0 + k;
                if (!vec && i >= e) continue;
                uint32_t w, code;
                unsigned long long cw;
                unit_of_code<SRC>(a, tab, i, codes[k], vec, unit, w, cw, code, bad_range);
                bits += w;
                zeros += (SRC == SRC_CODES && code == 0);
                if (w == 0 && (SRC != SRC_CODES || (tab && code < a.cap))) bad_width = true;
            }
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

// Exclusive scans over chunks (single CTA, 1024 threads): byte offsets
// (ceil(bits/8)) and outlier offsets.  Tiles of 4096 chunks are staged in
// shared memory with coalesced loads; each thread scans 4 consecutive entries.
__global__ void __cluster_dims__(kScanCtas, 1, 1) __launch_bounds__(1024) chunk_scan_kernel(DeflateArgs a) {
    cluster_chunk_scan(blockIdx.x, a.chunk_bits, a.chunk_zeros, a.nchunks, a.byte_off, a.out_off,
                       a.payload_cap, a.records != nullptr, a.out_cap, a.st);
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
    // a 1D block head: the dual-quant kept its prequantized value (no
    // scattered re-read of the input, one 128 B line per head)
    if (i < a.heads_limit && (i & 31) == 0) return a.heads[i >> 5];
    const void* p = a.in;
    uint64_t j = i;
    if (i >= a.in_split) { p = a.in_tail; j = i - a.in_split; }
    double v = a.in_kind == 0 ? (double)((const float*)p)[j] : ((const double*)p)[j];
    return a.in_kind == 2 ? v : prequant(v, two_eb);
}

// Per-warp bit-stream writer for one chunk.  Each call appends one <=64-bit
// left-aligned segment per lane, in lane order.  Output word j of the call
// is assembled by lane j % 32 from the few segments that overlap it: lanes
// mark the word whose first bit they cover, so the owner starts at the right
// segment without searching; no atomics, coalesced 32-bit stores.
struct WarpBitWriter {
    uint8_t* payload;
    uint64_t B, Bend;          // chunk byte range
    uint64_t wbyte;            // global byte address of the current word 0
    uint32_t carry_bits;       // bits already in carry_word
    uint32_t carry_word;
    unsigned long long* seg_s; // [32]
    uint32_t* off_s;           // [33]
    uint8_t* first_s;          // [68]

    __device__ __forceinline__ void emit(unsigned long long seg, uint32_t len, uint32_t lane) {
        int total_l;
        const uint32_t off = (uint32_t)warp_excl_scan((int)len, &total_l) + carry_bits;
        const uint32_t total = carry_bits + (uint32_t)total_l;
        seg_s[lane] = seg;
        off_s[lane] = off;
        if (lane == 31) off_s[32] = total;
        if (len) {
            uint32_t w = (off + 31) >> 5;                 // first word starting inside [off, off+len)
            if (32 * w < off + len) first_s[w] = (uint8_t)lane;
            if (32 * (w + 1) < off + len) first_s[w + 1] = (uint8_t)lane;
        }
        __syncwarp();
        const uint32_t nw = (total + 31) >> 5, full = total >> 5;
        uint32_t new_carry = 0;
        for (uint32_t j = lane; j < nw; j += 32) {
            const uint32_t ws = 32 * j, we = ws + 32;
            uint32_t word = j ? 0u : carry_word;
            for (uint32_t i = j ? first_s[j] : 0; i < 32; i++) {
                const uint32_t o = off_s[i];
                if (o >= we) break;
                if (off_s[i + 1] <= ws) continue;
                const unsigned long long sg = seg_s[i];
                word |= (o >= ws) ? ((uint32_t)(sg >> 32) >> (o - ws))
                                  : (uint32_t)((sg << (ws - o)) >> 32);
            }
            if (j < full) store_word(payload, wbyte + 4ull * j, word, B, Bend);
            else new_carry = word;
        }
        const uint32_t pc = __shfl_sync(kFull, new_carry, (nw - 1) & 31);
        __syncwarp();
        carry_word = (total & 31) ? pc : 0;
        wbyte += 4ull * full;
        carry_bits = total & 31;
    }
};

// pack: warp per chunk.  Lanes take 8 consecutive codes and build a <=64-bit
// segment (falling back to one code per lane per call when 8 codes overflow
// 64 bits); outliers (code 0) are compacted in row-major order.
template <int SRC, bool PAYLOAD, bool TS>
__global__ void __launch_bounds__(256) chunk_pack_kernel(DeflateArgs a) {
    extern __shared__ unsigned long long stable[];
    __shared__ unsigned long long s_seg[8][32];
    __shared__ uint32_t s_off[8][33];
    __shared__ uint8_t s_first[8][68];
    if (a.st->flags & (F_CODE_RANGE | F_ABSENT_SYM | F_ZERO_WIDTH | F_OVERFLOW | F_BW_TOO_BIG |
                       F_KRAFT | F_NO_PRESENT | F_ALL_ZERO_HIST))
        return;
    const uint32_t unit = unit_of(a);
    if (TS)
        for (uint32_t i = threadIdx.x; i < a.cap; i += blockDim.x) stable[i] = a.gtable[i];
    __syncthreads();
    const unsigned long long* tab = TS ? stable : a.gtable;
    const double two_eb = a.st->two_eb;
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    bool dummy = false;

    for (uint64_t c = blockIdx.x * 8ull + wid; c < a.nchunks; c += gridDim.x * 8ull) {
        const uint64_t s = c * a.chunk, e = umin(s + a.chunk, a.n);
        WarpBitWriter wr;
        wr.payload = a.payload;
        wr.B = a.byte_off[c];
        wr.Bend = wr.B + ((a.chunk_bits[c] + 7) >> 3);
        wr.wbyte = wr.B & ~3ull;
        wr.carry_bits = (uint32_t)(wr.B & 3) * 8;
        wr.carry_word = 0;
        wr.seg_s = s_seg[wid];
        wr.off_s = s_off[wid];
        wr.first_s = s_first[wid];
        uint64_t orec = a.out_off ? a.out_off[c] : 0;

        for (uint64_t g = s; g < e; g += 256) {
            const uint64_t i0 = g + 8 * lane;
            uint32_t codes[8];
            bool vec;
            load_group8<SRC>(a, i0, e, codes, vec);
            unsigned long long seg = 0;
            uint32_t len = 0, zc = 0;
            bool over = false;
            uint32_t code8[8];
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const uint64_t i = i0 + k;
                code8[k] = 1;
                if (!vec && i >= e) continue;
                uint32_t w, code;
                unsigned long long cw;
                unit_of_code<SRC>(a, tab, i, codes[k], vec, unit, w, cw, code, dummy);
                code8[k] = code;
                if (SRC == SRC_CODES && code == 0) zc++;
                if (len + w <= 64) {
                    if (w) seg |= cw << (64 - len - w);
                } else {
                    over = true;
                }
                len += w;
            }
            if (PAYLOAD) {
                if (!__any_sync(kFull, over)) {
                    wr.emit(seg, len, lane);
                } else {
                    for (int k = 0; k < 8; k++) {
                        const uint64_t i = g + 32 * k + lane;
                        unsigned long long sg = 0;
                        uint32_t w = 0;
                        if (i < e) {
                            uint32_t code;
                            unsigned long long cw;
                            fetch_unit<SRC>(a.src, tab, i, a.cap, unit, w, cw, code, dummy);
                            sg = w ? (cw << (64 - w)) : 0;
                        }
                        wr.emit(sg, w, lane);
                    }
                }
            }
            // outliers in row-major order
            if (SRC == SRC_CODES && a.records && __any_sync(kFull, zc)) {
                int ztot;
                uint32_t zoff = (uint32_t)warp_excl_scan((int)zc, &ztot);
                uint64_t slot = orec + zoff;
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const uint64_t i = i0 + k;
                    if (i < e && code8[k] == 0) {
                        if (i < a.rec_limit) {
                            const double v = outlier_value(a, i, two_eb);
                            a.records[2 * slot] = i + a.idx_base;
                            a.records[2 * slot + 1] = (unsigned long long)__double_as_longlong(v);
                        }
                        slot++;
                    }
                }
                orec += (uint64_t)ztot;
            }
        }
        if (PAYLOAD && wr.carry_bits && lane == 0)
            store_word(a.payload, wr.wbyte, wr.carry_word, wr.B, wr.Bend);
        __syncwarp();
    }
}

// --------------------------------------------------------------------------
// pack (fused path, uint16 codes): warp per chunk, rounds of 32 x kRun codes.
// Lane l owns the run of kRun consecutive codes [g + kRun*l, +kRun): pass A
// looks the codewords up (shared table) and sums their widths; one warp scan
// gives each run its bit offset; pass B streams the run MSB-first through a
// 64-bit accumulator into a per-warp shared word buffer.  Words strictly
// inside a run have a single writer (plain store); a run's first and last
// words are shared with its neighbours and merged with atomicOr (two per run,
// i.e. per 16 codes).  Completed words go to global memory coalesced; the
// trailing partial word carries into the next round.
// --------------------------------------------------------------------------
constexpr int kRun = 16;
constexpr int kRoundCodes = 32 * kRun;
constexpr int kBufWords = kRoundCodes * kMaxBw / 32 + 4;   // worst case 56 bits per code

// 32-bit units (every codeword <= 24 bits, the common case): the codebook is
// re-encoded as left-aligned codeword | width (width in the low 5 bits, which
// a <= 24-bit codeword leaves free), so appending a code is two funnel shifts
// into a 64-bit pending window; no 64-bit variable shifts, no branches.
__device__ __forceinline__ uint32_t entry32(unsigned long long u) {
    const uint32_t w = (uint32_t)(u >> 24);
    const uint32_t cw = (uint32_t)(u & 0xFFFFFFull);
    return w ? ((cw << (32 - w)) | w) : 0u;
}

__device__ __forceinline__ bool zero_half(uint32_t w) {   // either 16-bit half == 0
    return ((w - 0x00010001u) & ~w & 0x80008000u) != 0;
}

template <bool TS>
__global__ void __launch_bounds__(256, 3) chunk_pack32_kernel(DeflateArgs a) {
    __shared__ uint32_t s_tab[TS ? 4096 : 1];
    __shared__ uint32_t s_buf[8][kRoundCodes * 24 / 32 + 4];
    if (a.st->flags & (F_CODE_RANGE | F_ABSENT_SYM | F_ZERO_WIDTH | F_OVERFLOW | F_BW_TOO_BIG |
                       F_KRAFT | F_NO_PRESENT | F_ALL_ZERO_HIST))
        return;
    if (unit_of(a) != 32) return;   // 64-bit units: chunk_pack_run_kernel
    if (TS)
        for (uint32_t i = threadIdx.x; i < a.cap; i += blockDim.x) s_tab[i] = entry32(a.gtable[i]);
    __syncthreads();
    const double two_eb = a.st->two_eb;
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    uint32_t* buf = s_buf[wid];
    const uint16_t* src = (const uint16_t*)a.src;
    auto lookup = [&](uint32_t code) -> uint32_t {
        return TS ? s_tab[code] : entry32(__ldg(a.gtable + code));
    };
    for (uint64_t c = blockIdx.x * 8ull + wid; c < a.nchunks; c += gridDim.x * 8ull) {
        const uint64_t s = c * a.chunk, e = umin(s + a.chunk, a.n);
        const uint64_t B = a.byte_off[c];
        const uint64_t Bend = B + ((a.chunk_bits[c] + 7) >> 3);
        uint64_t wbyte = B & ~3ull;
        uint32_t carry = (uint32_t)(B & 3) * 8;
        uint32_t carry_word = 0;
        uint64_t orec = a.out_off ? a.out_off[c] : 0;
        // the next round's 16 codes per lane are in flight while this round packs
        auto fetch = [&](uint64_t g, uint4& v0, uint4& v1) -> bool {
            const uint64_t i0 = g + (uint64_t)kRun * lane;
            if (i0 + kRun > e || (i0 & 7)) return false;
            v0 = __ldg(reinterpret_cast<const uint4*>(src + i0));
            v1 = __ldg(reinterpret_cast<const uint4*>(src + i0) + 1);
            return true;
        };
        uint4 n0 = make_uint4(0, 0, 0, 0), n1 = n0;
        bool nvalid = fetch(s, n0, n1);
        for (uint64_t g = s; g < e; g += kRoundCodes) {
            const uint64_t i0 = g + (uint64_t)kRun * lane;
            const uint32_t cnt = i0 < e ? (uint32_t)umin(kRun, e - i0) : 0;
            const uint4 v0 = n0, v1 = n1;
            const bool valid = nvalid;
            nvalid = g + kRoundCodes < e && fetch(g + kRoundCodes, n0, n1);
            uint32_t code[kRun];
            bool anyz;
            if (valid) {
                const uint32_t wv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                anyz = false;
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    code[2 * k] = wv[k] & 0xFFFF;
                    code[2 * k + 1] = wv[k] >> 16;
                    anyz |= zero_half(wv[k]);
                }
            } else {
                anyz = false;
#pragma unroll
                for (int k = 0; k < kRun; k++) {
                    code[k] = (uint32_t)k < cnt ? src[i0 + k] : 1u;
                    anyz |= code[k] == 0;
                }
            }
            uint32_t ent[kRun], bits = 0;
            if (cnt == kRun) {
#pragma unroll
                for (int k = 0; k < kRun; k++) {
                    ent[k] = lookup(code[k]);
                    bits += ent[k] & 31u;
                }
            } else {
#pragma unroll
                for (int k = 0; k < kRun; k++) {
                    ent[k] = (uint32_t)k < cnt ? lookup(code[k]) : 0u;
                    bits += ent[k] & 31u;
                }
            }
            int total_l;
            const uint32_t off = (uint32_t)warp_excl_scan((int)bits, &total_l) + carry;
            const uint32_t total = carry + (uint32_t)total_l;
            // the previous round's trailing partial word seeds word 0
            if (lane == 0) buf[0] = carry_word;
#pragma unroll 1
            for (uint32_t j = lane + 1; j < (total + 31) >> 5; j += 32) buf[j] = 0;
            __syncwarp();
            // every codeword is OR-ed into the (at most two) words it touches:
            // no per-code branches or selects, one or two shared reductions
            {
                const uint32_t bufs = smem_u32(buf);
                uint32_t p = off;
#pragma unroll
                for (int k = 0; k < kRun; k++) {
                    const uint32_t al = ent[k] & ~31u, w = ent[k] & 31u;
                    const uint32_t sh = p & 31u, addr = bufs + ((p >> 5) << 2);
                    (void)w;
                    // the spill into the next word is 0 unless sh + w > 32, and
                    // w == 0 past a partial run: OR-ing 0 is harmless, so both
                    // reductions are unconditional (no branches)
                    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr), "r"(al >> sh) : "memory");
                    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr + 4), "r"(__funnelshift_r(0u, al, sh))
                                 : "memory");
                    p += w;
                }
            }
            __syncwarp();
            const uint32_t full = total >> 5;
            for (uint32_t j = lane; j < full; j += 32) store_word(a.payload, wbyte + 4ull * j, buf[j], B, Bend);
            carry_word = (total & 31) ? buf[full] : 0u;
            __syncwarp();
            wbyte += 4ull * full;
            carry = total & 31;
            // outliers (code 0) in row-major order
            if (a.records && __any_sync(kFull, anyz)) {
                uint32_t zc = 0;
#pragma unroll
                for (int k = 0; k < kRun; k++) zc += ((uint32_t)k < cnt) & (code[k] == 0);
                int ztot;
                const uint32_t zoff = (uint32_t)warp_excl_scan((int)zc, &ztot);
                uint64_t slot = orec + zoff;
#pragma unroll
                for (int k = 0; k < kRun; k++) {
                    if ((uint32_t)k < cnt && code[k] == 0) {
                        const uint64_t i = i0 + k;
                        if (i < a.rec_limit) {
                            const double v = outlier_value(a, i, two_eb);
                            a.records[2 * slot] = i + a.idx_base;
                            a.records[2 * slot + 1] = (unsigned long long)__double_as_longlong(v);
                        }
                        slot++;
                    }
                }
                orec += (uint64_t)ztot;
            }
        }
        if (carry && lane == 0) store_word(a.payload, wbyte, carry_word, B, Bend);
        __syncwarp();
    }
}

// --------------------------------------------------------------------------
// pack for long chunks (>= 32768 codes; 32-bit units): warp per chunk, rounds of
// 32 x Q x R codes.  Lane l owns Q consecutive sub-runs of R codes and shifts
// each sub-run's codewords into a 64-bit register (entry {width, codeword}:
// two funnel shifts, an OR and an add per code; no per-code shared traffic).
// One warp scan of the lane widths places every sub-run in the round's bit
// stream; a sub-run's left-aligned bits go to the <= 3 words of a per-warp
// shared buffer it touches: words whose first bit it holds by plain stores,
// then (after a warp sync) the word it starts inside of by one shared OR --
// every word has exactly one first-bit owner, so no zero fill is needed.
// Completed words go to global memory coalesced; the trailing partial word
// carries into the next round.  R is picked per chunk from its mean code
// length so a sub-run rarely exceeds 64 bits; one that does zeroes the words
// it owns and ORs its codewords in one by one.
// --------------------------------------------------------------------------
constexpr int kLaneCodes = 32;                             // Q x R codes per lane and round
constexpr int kPackBufWords = 32 * kLaneCodes * 24 / 32 + 4;   // 32-bit units: <= 24 bits per code

__device__ __forceinline__ uint32_t min_u16x2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

__device__ __forceinline__ void red_or(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t code_at(const uint32_t* wv, int k) {
    return (k & 1) ? (wv[k >> 1] >> 16) : (wv[k >> 1] & 0xFFFFu);
}

template <int R, int Q, bool TS>
__device__ __forceinline__ void pack32_chunk(const DeflateArgs& a, const uint2* s_tab, uint32_t* buf, uint64_t s,
                                             uint64_t e, uint64_t B, uint64_t Bend, uint64_t orec,
                                             double two_eb, uint32_t lane) {
    constexpr uint32_t LC = Q * R;       // codes per lane and round
    constexpr uint32_t RC = 32 * LC;     // codes per round
    static_assert(LC % 8 == 0 && LC <= kLaneCodes, "lane codes: whole 16-byte loads");
    const uint16_t* src = (const uint16_t*)a.src;
    auto lookup = [&](uint32_t code) -> uint2 {
        if (TS) return s_tab[code];
        const unsigned long long u = __ldg(a.gtable + code);
        return make_uint2((uint32_t)(u >> 24), (uint32_t)(u & 0xFFFFFFull));
    };
    const uint32_t bufs = smem_u32(buf);
    uint64_t wbyte = B & ~3ull;
    uint32_t carry = (uint32_t)(B & 3) * 8, carry_word = 0;
    bool first_round = true;
    // a lane's codes of the next round are in flight while this round packs
    // (16-byte loads when its run is whole and aligned)
    auto fetch = [&](uint64_t g, uint32_t (&wv)[LC / 2]) -> bool {
        const uint64_t i0 = g + (uint64_t)LC * lane;
        if (i0 + LC > e || (i0 & 7)) return false;
        const uint4* p = reinterpret_cast<const uint4*>(src + i0);
#pragma unroll
        for (int u = 0; u < (int)LC / 8; u++) {
            const uint4 v = __ldg(p + u);
            wv[4 * u] = v.x; wv[4 * u + 1] = v.y; wv[4 * u + 2] = v.z; wv[4 * u + 3] = v.w;
        }
        return true;
    };
    uint32_t nw[LC / 2];
#pragma unroll
    for (int k = 0; k < (int)LC / 2; k++) nw[k] = 0x00010001u;
    bool nvalid = fetch(s, nw);
    for (uint64_t g = s; g < e; g += RC) {
        const uint64_t i0 = g + (uint64_t)LC * lane;
        const uint32_t cnt = i0 < e ? (uint32_t)umin(LC, e - i0) : 0u;
        uint32_t wv[LC / 2];
#pragma unroll
        for (int k = 0; k < (int)LC / 2; k++) wv[k] = nw[k];
        const bool valid = nvalid;
        nvalid = g + RC < e && fetch(g + RC, nw);
        if (!valid) {   // ragged / unaligned run: scalar loads, past-the-end codes read as 1
#pragma unroll
            for (int k = 0; k < (int)LC; k += 2) {
                const uint32_t c0 = (uint32_t)k < cnt ? src[i0 + k] : 1u;
                const uint32_t c1 = (uint32_t)k + 1 < cnt ? src[i0 + k + 1] : 1u;
                wv[k >> 1] = c0 | (c1 << 16);
            }
        }
        // sub-runs in 64-bit registers, right-aligned, nb[q] bits (exact even past 64)
        uint32_t hi[Q] = {}, lo[Q] = {}, nb[Q] = {}, nbt = 0;
        auto append = [&](int q, uint2 t) {
            hi[q] = __funnelshift_l(lo[q], hi[q], t.x);
            lo[q] = __funnelshift_l(0u, lo[q], t.x) | t.y;
            nb[q] += t.x;
        };
        if (cnt == LC) {
#pragma unroll
            for (int k = 0; k < (int)LC; k++) append(k / R, lookup(code_at(wv, k)));
        } else {
#pragma unroll
            for (int k = 0; k < (int)LC; k++)
                append(k / R, ((uint32_t)k < cnt) ? lookup(code_at(wv, k)) : make_uint2(0u, 0u));
        }
#pragma unroll
        for (int q = 0; q < Q; q++) nbt += nb[q];
        int total_l;
        const uint32_t off = (uint32_t)warp_excl_scan((int)nbt, &total_l) + carry;
        const uint32_t total = carry + (uint32_t)total_l;
        // phase A: the words whose first bit a sub-run holds (the carry owns word 0's)
        if (lane == 0 && carry) sts32(bufs, carry_word);
        uint32_t Lh[Q], Ll[Q];
        {
            uint32_t o = off;
#pragma unroll
            for (int q = 0; q < Q; q++) {
                const uint32_t sh = o & 31u, a0 = bufs + ((o >> 5) << 2), end = o + nb[q];
                const uint32_t nxt = (o | 31u) + 1;   // first bit of the next word
                if (nb[q] <= 64) {
                    const uint32_t sl = 64 - nb[q];   // left-align
                    Lh[q] = sl >= 32 ? lo[q] << (sl - 32) : __funnelshift_l(lo[q], hi[q], sl);
                    Ll[q] = sl >= 32 ? 0u : lo[q] << sl;
                    if (sh == 0 && nb[q]) sts32(a0, Lh[q]);
                    if (nxt < end) sts32(a0 + 4, __funnelshift_r(Ll[q], Lh[q], sh));
                    if (nxt + 32 < end) sts32(a0 + 8, __funnelshift_r(0u, Ll[q], sh));
                } else {   // longer than 64 bits: zero the owned words, OR codewords in below
                    for (uint32_t j = (o + 31) >> 5; 32 * j < end; j++) sts32(bufs + 4 * j, 0u);
                }
                o = end;
            }
        }
        __syncwarp();
        // phase B: the word each sub-run starts inside of
        {
            uint32_t o = off;
#pragma unroll
            for (int q = 0; q < Q; q++) {
                const uint32_t sh = o & 31u, a0 = bufs + ((o >> 5) << 2);
                if (nb[q] <= 64) {
                    if (sh && nb[q]) red_or(a0, Lh[q] >> sh);
                } else {
                    uint32_t p = o;
#pragma unroll
                    for (int k = q * R; k < (q + 1) * R; k++) {
                        const uint2 t = ((uint32_t)k < cnt) ? lookup(code_at(wv, k)) : make_uint2(0u, 0u);
                        if (t.x) {
                            const uint32_t al = t.y << (32 - t.x);
                            const uint32_t ps = p & 31u, pa = bufs + ((p >> 5) << 2);
                            red_or(pa, al >> ps);
                            if (ps + t.x > 32) red_or(pa + 4, __funnelshift_r(0u, al, ps));
                            p += t.x;
                        }
                    }
                }
                o += nb[q];
            }
        }
        __syncwarp();
        const uint32_t full = total >> 5;
        for (uint32_t j = lane; j < full; j += 32) {
            const uint32_t w = buf[j];
            if (j == 0 && first_round) store_word(a.payload, wbyte, w, B, Bend);   // may start before B
            else *reinterpret_cast<uint32_t*>(a.payload + wbyte + 4ull * j) = bswap32(w);
        }
        carry_word = (total & 31) ? buf[full] : 0u;
        __syncwarp();
        wbyte += 4ull * full;
        carry = total & 31;
        first_round = first_round && full == 0;
        // outliers (code 0) in row-major order
        if (a.records) {
            uint32_t m = wv[0];
#pragma unroll
            for (int k = 1; k < (int)LC / 2; k++) m = min_u16x2(m, wv[k]);
            const bool anyz = cnt != 0 && zero_half(m);
            if (__any_sync(kFull, anyz)) {
                uint32_t zc = 0;
#pragma unroll
                for (int k = 0; k < (int)LC; k++) zc += ((uint32_t)k < cnt) & (code_at(wv, k) == 0);
                int ztot;
                const uint32_t zoff = (uint32_t)warp_excl_scan((int)zc, &ztot);
                uint64_t slot = orec + zoff;
#pragma unroll
                for (int k = 0; k < (int)LC; k++) {
                    if ((uint32_t)k < cnt && code_at(wv, k) == 0) {
                        const uint64_t i = i0 + k;
                        if (i < a.rec_limit) {
                            const double v = outlier_value(a, i, two_eb);
                            a.records[2 * slot] = i + a.idx_base;
                            a.records[2 * slot + 1] = (unsigned long long)__double_as_longlong(v);
                        }
                        slot++;
                    }
                }
                orec += (uint64_t)ztot;
            }
        }
    }
    if (carry && lane == 0) store_word(a.payload, wbyte, carry_word, B, Bend);
    __syncwarp();
}

constexpr size_t kPack32Smem = 4096 * sizeof(uint2) + 8 * kPackBufWords * 4;

template <bool TS>
__global__ void __launch_bounds__(256, 2) chunk_pack32_runs_kernel(DeflateArgs a) {
    extern __shared__ __align__(16) unsigned char pack_smem[];
    uint2* s_tab = reinterpret_cast<uint2*>(pack_smem);
    uint32_t* s_buf = reinterpret_cast<uint32_t*>(pack_smem + (TS ? 4096 * sizeof(uint2) : 0));
    if (a.st->flags & (F_CODE_RANGE | F_ABSENT_SYM | F_ZERO_WIDTH | F_OVERFLOW | F_BW_TOO_BIG |
                       F_KRAFT | F_NO_PRESENT | F_ALL_ZERO_HIST))
        return;
    if (unit_of(a) != 32) return;   // 64-bit units: chunk_pack_run_kernel
    if (TS)
        for (uint32_t i = threadIdx.x; i < a.cap; i += blockDim.x) {
            const unsigned long long u = a.gtable[i];
            s_tab[i] = make_uint2((uint32_t)(u >> 24), (uint32_t)(u & 0xFFFFFFull));
        }
    __syncthreads();
    const double two_eb = a.st->two_eb;
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    uint32_t* buf = s_buf + wid * kPackBufWords;
    for (uint64_t c = blockIdx.x * 8ull + wid; c < a.nchunks; c += gridDim.x * 8ull) {
        const uint64_t s = c * a.chunk, e = umin(s + a.chunk, a.n);
        const uint32_t bits = a.chunk_bits[c];
        const uint64_t B = a.byte_off[c];
        const uint64_t Bend = B + ((bits + 7) >> 3);
        const uint64_t orec = a.out_off ? a.out_off[c] : 0;
        // sub-runs of ~44 bits at the chunk's mean code length
        const uint64_t len = e - s;
        if (16ull * bits <= 44ull * len)
            pack32_chunk<16, 2, TS>(a, s_tab, buf, s, e, B, Bend, orec, two_eb, lane);
        else if (8ull * bits <= 44ull * len)
            pack32_chunk<8, 4, TS>(a, s_tab, buf, s, e, B, Bend, orec, two_eb, lane);
        else
            pack32_chunk<4, 4, TS>(a, s_tab, buf, s, e, B, Bend, orec, two_eb, lane);
    }
}

template <bool TS>
__global__ void __launch_bounds__(256) chunk_pack_run_kernel(DeflateArgs a, int want_payload) {
    extern __shared__ unsigned long long stable[];
    __shared__ uint32_t s_buf[8][kBufWords];
    if (a.st->flags & (F_CODE_RANGE | F_ABSENT_SYM | F_ZERO_WIDTH | F_OVERFLOW | F_BW_TOO_BIG |
                       F_KRAFT | F_NO_PRESENT | F_ALL_ZERO_HIST))
        return;
    const uint32_t unit = unit_of(a);
    const bool payload = want_payload != 0 && a.gtable != nullptr;
    if (payload && unit == 32) return;   // chunk_pack32_kernel packs it
    const uint32_t wshift = unit - 8;
    const unsigned long long cwmask = (1ull << wshift) - 1;
    if (TS)
        for (uint32_t i = threadIdx.x; i < a.cap; i += blockDim.x) stable[i] = a.gtable[i];
    __syncthreads();
    const unsigned long long* tab = TS ? stable : a.gtable;
    const double two_eb = a.st->two_eb;
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    uint32_t* buf = s_buf[wid];
    const uint16_t* src = (const uint16_t*)a.src;

    for (uint64_t c = blockIdx.x * 8ull + wid; c < a.nchunks; c += gridDim.x * 8ull) {
        const uint64_t s = c * a.chunk, e = umin(s + a.chunk, a.n);
        const uint64_t B = a.byte_off[c];
        const uint64_t Bend = B + ((a.chunk_bits[c] + 7) >> 3);
        uint64_t wbyte = B & ~3ull;
        uint32_t carry = (uint32_t)(B & 3) * 8;
        uint64_t orec = a.out_off ? a.out_off[c] : 0;
        for (uint32_t i = lane; i < kBufWords; i += 32) buf[i] = 0;
        __syncwarp();
        for (uint64_t g = s; g < e; g += kRoundCodes) {
            const uint64_t i0 = g + (uint64_t)kRun * lane;
            const uint32_t cnt = i0 < e ? (uint32_t)umin(kRun, e - i0) : 0;
            // pass A: codes, widths, zero count
            uint32_t code[kRun];
            if (cnt == kRun && (i0 & 7) == 0) {
                const uint4 v0 = __ldg(reinterpret_cast<const uint4*>(src + i0));
                const uint4 v1 = __ldg(reinterpret_cast<const uint4*>(src + i0) + 1);
                const uint32_t wv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    code[2 * k] = wv[k] & 0xFFFF;
                    code[2 * k + 1] = wv[k] >> 16;
                }
            } else {
#pragma unroll
                for (int k = 0; k < kRun; k++) code[k] = (uint32_t)k < cnt ? src[i0 + k] : 1u;
            }
            uint32_t bits = 0, zc = 0;
            unsigned long long u[kRun];
#pragma unroll
            for (int k = 0; k < kRun; k++) {
                u[k] = ((uint32_t)k < cnt && payload) ? tab[code[k]] : 0ull;
                bits += (uint32_t)(u[k] >> wshift);
                zc += ((uint32_t)k < cnt) & (code[k] == 0);
            }
            int total_l;
            const uint32_t off = (uint32_t)warp_excl_scan((int)bits, &total_l) + carry;
            const uint32_t total = carry + (uint32_t)total_l;
            // pass B: stream the run into the word buffer.  Branch-free: a
            // completed word is a predicated plain store, except the run's
            // first and last words, which neighbouring runs share and which are
            // OR-ed in after the loop (two shared atomics per 16 codes).
            if (payload && bits) {
                uint32_t wi = off >> 5;
                uint32_t nacc = off & 31;            // leading bits belong to earlier runs
                unsigned long long acc = 0;          // left-aligned pending bits
                const uint32_t wfirst = wi;
                uint32_t first_word = 0;
                bool have_first = false;
#pragma unroll
                for (int k = 0; k < kRun; k++) {
                    uint32_t w = (uint32_t)(u[k] >> wshift);
                    unsigned long long cw = u[k] & cwmask;
                    if (unit > 32 && w > 32) {       // 64-bit units: emit the high part first
                        const uint32_t wh = w - 32;
                        acc |= (cw >> 32) << (64 - nacc - wh);
                        nacc += wh;
                        cw &= 0xFFFFFFFFull;
                        w = 32;
                        if (nacc >= 32) {
                            const uint32_t word = (uint32_t)(acc >> 32);
                            if (have_first) buf[wi] = word; else first_word = word;
                            have_first = true;
                            wi++;
                            acc <<= 32;
                            nacc -= 32;
                        }
                    }
                    acc |= w ? (cw << (64 - nacc - w)) : 0ull;
                    nacc += w;
                    const bool emit = nacc >= 32;
                    const uint32_t word = (uint32_t)(acc >> 32);
                    if (emit && have_first) buf[wi] = word;
                    first_word = (emit && !have_first) ? word : first_word;
                    have_first |= emit;
                    wi += emit ? 1u : 0u;
                    acc = emit ? (acc << 32) : acc;
                    nacc -= emit ? 32u : 0u;
                }
                // (the shared ORs below are atomic: no ordering against the
                // neighbours' plain stores is needed -- those words differ)
                if (have_first) atomicOr(&buf[wfirst], first_word);
                if (nacc) atomicOr(&buf[wi], (uint32_t)(acc >> 32));
            }
            __syncwarp();
            if (payload) {
                const uint32_t full = total >> 5;
                for (uint32_t j = lane; j < full; j += 32) store_word(a.payload, wbyte + 4ull * j, buf[j], B, Bend);
                __syncwarp();
                const uint32_t used = (total + 31) >> 5;
                const uint32_t cw_last = (total & 31) ? buf[full] : 0u;
                __syncwarp();   // every lane has read the carry word before it is cleared
                for (uint32_t j = lane; j < used; j += 32) buf[j] = 0;
                __syncwarp();
                if (lane == 0) buf[0] = cw_last;
                __syncwarp();
                wbyte += 4ull * full;
                carry = total & 31;
            }
            // outliers (code 0) in row-major order
            if (a.records && __any_sync(kFull, zc)) {
                int ztot;
                const uint32_t zoff = (uint32_t)warp_excl_scan((int)zc, &ztot);
                uint64_t slot = orec + zoff;
#pragma unroll
                for (int k = 0; k < kRun; k++) {
                    if ((uint32_t)k < cnt && code[k] == 0) {
                        const uint64_t i = i0 + k;
                        if (i < a.rec_limit) {
                            const double v = outlier_value(a, i, two_eb);
                            a.records[2 * slot] = i + a.idx_base;
                            a.records[2 * slot + 1] = (unsigned long long)__double_as_longlong(v);
                        }
                        slot++;
                    }
                }
                orec += (uint64_t)ztot;
            }
        }
        if (payload && carry && lane == 0) store_word(a.payload, wbyte, buf[0], B, Bend);
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

// MSB-first bit reader over the payload with a software-pipelined 16-byte
// prefetch: the block after the one being consumed is always in flight, so
// the ~1 us global-load latency is hidden behind ~40 decoded codewords and
// never stalls the lockstep warp (one lane refilling would stall all 32).
struct BitReader {
    const uint4* blk;
    uint64_t nblk;                 // readable 16 B blocks (payload + zero padding)
    unsigned long long buf;        // left-aligned valid bits
    int nb;
    unsigned long long qhi, qlo;   // queued big-endian words
    int qw;
    uint4 nxt;                     // prefetched block
    uint64_t next_idx;

    __device__ __forceinline__ uint4 load(uint64_t i) const {
        return i < nblk ? __ldg(blk + i) : make_uint4(0, 0, 0, 0);
    }
    __device__ __forceinline__ void take(const uint4& v) {
        qhi = ((unsigned long long)bswap32(v.x) << 32) | bswap32(v.y);
        qlo = ((unsigned long long)bswap32(v.z) << 32) | bswap32(v.w);
        qw = 4;
    }
    __device__ __forceinline__ uint32_t pop() {
        if (qw == 0) {
            take(nxt);
            nxt = load(next_idx++);
        }
        uint32_t w = (uint32_t)(qhi >> 32);
        qhi = (qhi << 32) | (qlo >> 32);
        qlo <<= 32;
        qw--;
        return w;
    }
    __device__ __forceinline__ void refill() {   // steady state: nb > 0, one pop suffices
        if (nb <= 32) {
            buf |= (unsigned long long)pop() << (32 - nb);
            nb += 32;
        }
    }
    __device__ __forceinline__ void init(uint64_t bit) {
        uint64_t b = bit >> 7;
        take(load(b));
        nxt = load(b + 1);
        next_idx = b + 2;
        uint32_t off = (uint32_t)(bit & 127);
        for (uint32_t s = 0; s < (off >> 5); s++) pop();
        buf = 0;
        nb = 0;
        refill();
        refill();
        uint32_t sh = off & 31;
        buf <<= sh;
        nb -= (int)sh;
        refill();
    }
    __device__ __forceinline__ void skip(uint32_t len) {
        buf = len < 64 ? (buf << len) : 0;
        nb -= (int)len;
    }
};

template <bool OUT32>
__global__ void __launch_bounds__(64) inflate_kernel(
    const uint8_t* __restrict__ payload, uint64_t nwords, const uint32_t* __restrict__ chunk_bits,
    const unsigned long long* __restrict__ byte_off, uint64_t nchunks, uint32_t chunk, uint64_t n,
    const uint64_t* __restrict__ gfirst, const int64_t* __restrict__ goffsets,
    const uint32_t* __restrict__ symbols, const uint32_t* __restrict__ glut, int max_bw_arg,
    void* out, DevStatus* st, const uint8_t* __restrict__ only) {
    // `only` != null: decode just the chunks the warp-parallel decoder handed
    // back (tiny chunks, corrupt streams -> exact reference error semantics)
    const uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (only && st->pad[1] == 0) return;   // the warp-parallel decoder handed nothing back (CTA-uniform)
    // a CTA whose chunks were all decoded by the warp-parallel decoder has nothing to do
    if (!__syncthreads_or(!only || (c < nchunks && only[c]))) return;
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
    uint32_t zeros = 0;
    if (c < nchunks && (!only || only[c])) {
        if (only) atomicAdd(&st->pad[2], 1ull);   // diagnostics: chunks handed back
        const uint32_t* words = reinterpret_cast<const uint32_t*>(payload);
        const uint64_t sbit = byte_off[c] * 8;
        const uint32_t budget = chunk_bits[c];
        const uint64_t base = c * chunk;
        const uint64_t cnt = umin(chunk, n - base);
        const bool vec = !OUT32 && (base & 7) == 0;
        uint16_t* out16 = (uint16_t*)out + base;
        BitReader rd;
        rd.blk = reinterpret_cast<const uint4*>(payload);
        rd.nblk = nwords / 4;
        rd.init(sbit);
        uint32_t pos = 0;
        unsigned long long err = ~0ull;
        unsigned long long acc0 = 0, acc1 = 0;   // 8 pending uint16 codes
        uint64_t k = 0;
        for (; k < cnt; k++) {
            rd.refill();
            uint32_t e = lut[rd.buf >> (64 - lb)];
            uint32_t len = (e >> 16) & 0xFF;
            uint32_t sym = e & 0xFFFF;
            if (len == 0) {
                // canonical search beyond the LUT (huffman.py:295-305)
                uint64_t p = sbit + pos;
                uint64_t pw = p >> 5;
                uint32_t ps = (uint32_t)(p & 31);
                unsigned long long hi64 = ((unsigned long long)load_be(words, pw, nwords) << 32) |
                                          load_be(words, pw + 1, nwords);
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
            zeros += (sym == 0);
            pos += len;
            if (OUT32) {
                ((uint32_t*)out)[base + k] = sym;
            } else if (vec) {
                const uint32_t j = (uint32_t)(k & 7);
                if (j < 4) acc0 |= (unsigned long long)sym << (16 * j);
                else acc1 |= (unsigned long long)sym << (16 * (j - 4));
                if (j == 7) {
                    *reinterpret_cast<uint4*>(out16 + k - 7) =
                        make_uint4((uint32_t)acc0, (uint32_t)(acc0 >> 32), (uint32_t)acc1,
                                   (uint32_t)(acc1 >> 32));
                    acc0 = acc1 = 0;
                }
            } else {
                out16[k] = (uint16_t)sym;
            }
            if ((int)len <= rd.nb) rd.skip(len);
            else rd.init(sbit + pos);   // a codeword longer than the window: resync
        }
        if (vec && err == ~0ull) {
            for (uint64_t j = k & ~7ull; j < k; j++) {
                uint32_t t = (uint32_t)(j & 7);
                out16[j] = (uint16_t)((t < 4 ? acc0 >> (16 * t) : acc1 >> (16 * (t - 4))) & 0xFFFF);
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
    const bool ts = SRC == SRC_CODES && a.gtable && a.cap <= 4096;
    size_t smem = ts ? a.cap * 8 : 0;
    uint64_t grid = ceil_div(a.nchunks, 8);
    if (grid > (uint64_t)ctx->num_sms * 16) grid = ctx->num_sms * 16;
    if (grid < 1) grid = 1;
    if (SRC == SRC_CODES && a.gtable && a.trusted && a.cap <= 4096) {
        chunk_stats_fast_kernel<<<(unsigned)grid, 256, 0, ctx->stream>>>(a);
        SDQZ_LAUNCHED_NAMED(ctx, "chunk_stats_kernel");
    } else {
        if (ts) chunk_stats_kernel<SRC, true><<<(unsigned)grid, 256, smem, ctx->stream>>>(a);
        else chunk_stats_kernel<SRC, false><<<(unsigned)grid, 256, 0, ctx->stream>>>(a);
        SDQZ_LAUNCHED_NAMED(ctx, "chunk_stats_kernel");
    }
    chunk_scan_kernel<<<kScanCtas, 1024, 0, ctx->stream>>>(a);
    SDQZ_LAUNCHED_NAMED(ctx, "chunk_scan_kernel");
    if (SRC == SRC_CODES) {
        // 28.8 KB static + up to 32 KB table > the 48 KB default
        ensure_smem(ctx, (const void*)chunk_pack_run_kernel<true>, 4096 * 8);
        if (payload && a.gtable) {   // 32-bit units (device-decided; no-op otherwise)
            static const uint32_t runs_min = [] {   // SDQZ_PACK_RUNS_MIN: tuning override
                const char* e = getenv("SDQZ_PACK_RUNS_MIN");
                return e ? (uint32_t)atoi(e) : 32768u;
            }();
            if (a.chunk >= runs_min) {   // long chunks: register runs (amortise the per-round warp work)
                ensure_smem(ctx, (const void*)chunk_pack32_runs_kernel<true>, kPack32Smem);
                ensure_smem(ctx, (const void*)chunk_pack32_runs_kernel<false>, 8 * kPackBufWords * 4);
                if (ts) chunk_pack32_runs_kernel<true><<<(unsigned)grid, 256, kPack32Smem, ctx->stream>>>(a);
                else chunk_pack32_runs_kernel<false><<<(unsigned)grid, 256, 8 * kPackBufWords * 4, ctx->stream>>>(a);
            } else if (ts) {
                chunk_pack32_kernel<true><<<(unsigned)grid, 256, 0, ctx->stream>>>(a);
            } else {
                chunk_pack32_kernel<false><<<(unsigned)grid, 256, 0, ctx->stream>>>(a);
            }
            SDQZ_LAUNCHED_NAMED(ctx, "chunk_pack32_kernel");
        }
        // 64-bit units (or no payload): device-decided, usually an idle launch;
        // two CTAs per SM walk the chunks
        const unsigned rgrid = (unsigned)umin(grid, (uint64_t)ctx->num_sms * 2);
        if (ts) chunk_pack_run_kernel<true><<<rgrid, 256, smem, ctx->stream>>>(a, payload ? 1 : 0);
        else chunk_pack_run_kernel<false><<<rgrid, 256, 0, ctx->stream>>>(a, payload ? 1 : 0);
    } else {
        chunk_pack_kernel<SRC, true, false><<<(unsigned)grid, 256, 0, ctx->stream>>>(a);
    }
    SDQZ_LAUNCHED_NAMED(ctx, "chunk_pack_kernel");
    return SDQZ_OK;
}

}  // namespace

int launch_histogram_u32(sdqz_ctx* ctx, const uint32_t* codes, uint64_t n, uint32_t cap,
                         unsigned long long* hist) {
    size_t smem = cap <= 16384 ? cap * 4 : 0;
    ensure_smem(ctx, (const void*)hist_u32_kernel, smem);
    uint64_t grid = ceil_div(n, 256);
    if (grid > (uint64_t)ctx->num_sms * 4) grid = ctx->num_sms * 4;
    if (grid < 1) grid = 1;
    hist_u32_kernel<<<(unsigned)grid, 256, smem, ctx->stream>>>(codes, n, cap, hist, ctx->d_status);
    SDQZ_LAUNCHED_NAMED(ctx, "hist_u32_kernel");
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
    // static shared memory (~17 KB) + dynamic can pass 48 KB
    ensure_smem(ctx, (const void*)codebook_kernel<true>, smem);
    static const uint32_t round_min = [] {
        const char* e = getenv("SDQZ_ROUND_MIN");
        const uint32_t r = e ? (uint32_t)atoi(e) : 4u;
        return r ? r : 1u;
    }();
    if (cap <= kSmemSortMax)
        codebook_kernel<true><<<1, kBookThreads, smem, ctx->stream>>>(d_hist, d_bw, cap, book, ctx->d_status,
                                                                   build_tree ? 1 : 0, canon ? 1 : 0, gs,
                                                                   round_min);
    else
        codebook_kernel<false><<<1, kBookThreads, 0, ctx->stream>>>(d_hist, d_bw, cap, book, ctx->d_status,
                                                                    build_tree ? 1 : 0, canon ? 1 : 0, gs,
                                                                    round_min);
    SDQZ_LAUNCHED_NAMED(ctx, "codebook_kernel");
    return SDQZ_OK;
}

int launch_build_lut(sdqz_ctx* ctx, const uint64_t* first, const int64_t* offsets,
                     const uint32_t* symbols, int max_bw_or_neg, uint32_t* lut) {
    lut_kernel<<<16, 256, 0, ctx->stream>>>(first, offsets, symbols, max_bw_or_neg, ctx->d_status, lut);
    SDQZ_LAUNCHED_NAMED(ctx, "lut_kernel");
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
    a.rec_limit = job.rec_limit;
    a.records = (unsigned long long*)job.out_records;
    a.out_cap = job.out_cap;
    a.heads = job.heads;
    a.heads_limit = job.heads ? job.heads_limit : 0;
    a.trusted = job.trusted;
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
    SDQZ_LAUNCHED_NAMED(ctx, "encode_kernel");
    return SDQZ_OK;
}

int launch_inflate(sdqz_ctx* ctx, const uint8_t* payload, uint64_t payload_bytes,
                   const uint32_t* chunk_bits, uint64_t n_chunks, uint32_t chunk,
                   const uint64_t* first, const int64_t* offsets, const uint32_t* symbols,
                   const uint32_t* lut, int max_bw, uint32_t cap, uint64_t n, void* codes, bool out32,
                   uint64_t stream_bytes) {
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
    uint64_t grid = ceil_div(n_chunks, 64);
    if (out32) {
        chunk_scan_kernel<<<kScanCtas, 1024, 0, ctx->stream>>>(a);
        SDQZ_LAUNCHED_NAMED(ctx, "chunk_scan_kernel");
        inflate_kernel<true><<<(unsigned)grid, 64, 0, ctx->stream>>>(
            payload, nwords, chunk_bits, a.byte_off, n_chunks, chunk, n, first, offsets, symbols, lut,
            max_bw, codes, ctx->d_status, nullptr);
        SDQZ_LAUNCHED_NAMED(ctx, "inflate_kernel");
        return SDQZ_OK;
    }
    // warp-parallel decode; chunks it hands back are redone sequentially
    uint8_t* redo = scratch_as<uint8_t>(ctx, S_REDO, n_chunks, &rc);
    if (!redo) return rc;
    // one launch: decode tables (+ the fallback LUT) | chunk byte offsets + clears
    (void)cap;
    uint32_t* tab = nullptr;
    // table width from the stream's mean code length (its own size, not the buffer's)
    const int ns = decode_ns(stream_bytes ? stream_bytes : payload_bytes, n);
    if ((rc = launch_decode_prep(ctx, first, offsets, symbols, max_bw, &tab, const_cast<uint32_t*>(lut),
                                 chunk_bits, n_chunks, a.byte_off, redo, ns)))
        return rc;
    if ((rc = launch_inflate_fast(ctx, payload, nwords, chunk_bits, a.byte_off, n_chunks, chunk, n,
                                  first, offsets, symbols, tab, max_bw, (uint16_t*)codes, redo, ns)))
        return rc;
    inflate_kernel<false><<<(unsigned)grid, 64, 0, ctx->stream>>>(
        payload, nwords, chunk_bits, a.byte_off, n_chunks, chunk, n, first, offsets, symbols, lut,
        max_bw, codes, ctx->d_status, redo);
    SDQZ_LAUNCHED_NAMED(ctx, "inflate_kernel");
    return SDQZ_OK;
}

}  // namespace sdqz
