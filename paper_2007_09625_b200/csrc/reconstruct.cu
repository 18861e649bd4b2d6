// reconstruct.cu -- K6: reversed dual-quantization (dualquant.py:197-227,
// :276-332) as exact integer prefix sums.
//
// Within a block the Lorenzo inverse is final = P_x P_y P_z delta', where
// delta' is the residual field with the (unknown) true residual at each
// outlier.  Streaming over planes z and rows y with lane = x:
//     final(z,y,x) = u(x) + K(x),  K = f(z,y-1,x) + f(z-1,y,x) - f(z-1,y-1,x),
//     u = P_x delta'  (segmented warp scan over the block's 8 / 16 / 32 lanes).
// An outlier at p carries its final value v, so u(p) = v - K(p); to its right
// (up to the next outlier) u(x) = S(x) - S(p) + v - K(p) with S = scan of the
// in-cap residuals.  Each lane therefore takes the correction t = v - K - S of
// the last outlier at or left of it in its segment (ballot + shuffle): O(1)
// per point, no per-outlier loop, exact in int64.
//
// Outlier values come straight from the archive's sorted records: a zero code
// at flat index i (code 0 <=> outlier, validated) finds its record in the
// 1024-point bucket i/1024 of a bucket table (OutLookup, one probe where the
// records are evenly spread, else a short binary search) -- no dense side
// array.  A block whose outlier values are not integers below 2^40 (the int64
// path would no longer match fp64 rounding) is flagged and redone by a generic
// kernel that replays the reference's fp64 operation order exactly (cumsum per
// axis, then per-outlier box corrections in raster order); non-default block
// shapes run the thread-per-block rq_blocks_kernel.
#include "kernels.cuh"

namespace sdqz {

namespace {

constexpr int kThreads = 256;
constexpr int kWarpsPerCta = kThreads / 32;
constexpr double kExact = 1099511627776.0;   // 2^40
constexpr uint64_t kSlotPts = 512;            // per-thread replay slot (largest fast block shape)

struct Geo {
    int nd;
    uint64_t dims[3];
    uint32_t block[3];
    uint64_t stride[3];
    uint64_t nblk[3];
};

__device__ __forceinline__ uint64_t block_of(const Geo& g, uint64_t idx) {
    uint64_t rem = idx, b = 0;
    for (int a = 0; a < g.nd; a++) {
        uint64_t c = rem / g.stride[a];
        rem -= c * g.stride[a];
        b = b * g.nblk[a] + c / g.block[a];
    }
    return b;
}

__global__ void outlier_scatter_kernel(const unsigned long long* __restrict__ rec,
                                       const uint64_t* __restrict__ idxs, const double* __restrict__ vals,
                                       uint64_t k, uint64_t n, const uint16_t* __restrict__ codes, Geo g,
                                       uint8_t* blockflag,
                                       DevStatus* st, int check_only) {
    // check_only (1D records path): order / range / fp64-path checks; the
    // codes[idx] == 0 check and the outlier values are taken by the
    // reconstruct kernel from the records, so only the records of a flagged
    // (fp64-path) block are scattered, for rq_generic_kernel
    unsigned long long f = 0;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < k;
         j += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t idx = rec ? rec[2 * j] : idxs[j];
        unsigned long long vb = rec ? rec[2 * j + 1] : (unsigned long long)__double_as_longlong(vals[j]);
        if (j > 0) {
            uint64_t prev = rec ? rec[2 * (j - 1)] : idxs[j - 1];
            if ((long long)idx - (long long)prev <= 0) f |= F_OUT_ORDER;
        }
        if (idx >= n) { f |= F_OUT_RANGE; continue; }
        if (!check_only && codes[idx] != 0) f |= F_OUT_NONZERO;
        double v = __longlong_as_double((long long)vb);
        if (!(fabs(v) < kExact && v == floor(v))) {
            blockflag[block_of(g, idx)] = 1;
            f |= F_OUT_SLOW;
        }
    }
    if (f) atomicOr(&st->flags, f);
}

__global__ void count_zero_kernel(const uint16_t* __restrict__ codes, uint64_t n, DevStatus* st) {
    uint32_t z = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        z += codes[i] == 0;
    z = __reduce_add_sync(kFull, z);
    if (lane_id() == 0 && z) atomicAdd(&st->n_zero, (unsigned long long)z);
}

__global__ void narrow_codes_kernel(const uint32_t* __restrict__ in, uint64_t n, uint32_t cap,
                                    uint16_t* __restrict__ out, DevStatus* st) {
    bool bad = false;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c = in[i];
        if (c >= cap) { bad = true; c = 1; }
        out[i] = (uint16_t)c;
    }
    if (bad) atomicOr(&st->flags, (unsigned long long)F_CODE_RANGE);
}

template <int OUTK>
__device__ __forceinline__ void store_out(void* out, uint64_t i, long long fin, double two_eb) {
    double v = __dmul_rn((double)fin, two_eb);
    if (OUTK == 0) ((float*)out)[i] = __double2float_rn(v);
    else ((double*)out)[i] = v;
}

// fused quality (metrics.py:52-76): per-thread partials of the stored values
// against the original field, folded per CTA into part[blockIdx.x]
struct QAcc {
    double ss = 0.0, mx = 0.0, mn = INFINITY, mo = -INFINITY;
    bool bad = false;
    __device__ __forceinline__ void add(const QualArgs& q, uint64_t i, double y) {
        const double x = q.okind ? __ldcs((const double*)q.orig + i) : (double)__ldcs((const float*)q.orig + i);
        const double d = __dsub_rn(x, y);
        ss = __fma_rn(d, d, ss);
        mx = isnan(d) ? d : fmax(mx, fabs(d));
        mn = fmin(mn, x);
        mo = fmax(mo, x);
        bad |= !isfinite(x);
    }
};

// block reduction of the partials (every thread of the CTA calls it once)
__device__ void qacc_flush(QAcc& a, const QualArgs& q) {
    __shared__ double s[5][32];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        a.ss += __shfl_down_sync(kFull, a.ss, o);
        const double m2 = __shfl_down_sync(kFull, a.mx, o);
        a.mx = isnan(m2) ? m2 : fmax(a.mx, m2);
        a.mn = fmin(a.mn, __shfl_down_sync(kFull, a.mn, o));
        a.mo = fmax(a.mo, __shfl_down_sync(kFull, a.mo, o));
    }
    const bool wbad = __any_sync(kFull, a.bad);
    if (lane == 0) { s[0][w] = a.ss; s[1][w] = a.mx; s[2][w] = a.mn; s[3][w] = a.mo; s[4][w] = wbad ? 1.0 : 0.0; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double r0 = 0.0, r1 = 0.0, r2 = INFINITY, r3 = -INFINITY, r4 = 0.0;
        for (uint32_t k = 0; k < nw; k++) {
            r0 += s[0][k];
            r1 = isnan(s[1][k]) ? s[1][k] : fmax(r1, s[1][k]);
            r2 = fmin(r2, s[2][k]);
            r3 = fmax(r3, s[3][k]);
            r4 = fmax(r4, s[4][k]);
        }
        double* p = q.part + 5 * blockIdx.x;
        p[0] = r0; p[1] = r1; p[2] = r2; p[3] = r3; p[4] = r4;
    }
}

// f64 bits of the record at flat index i (0 when there is none: only for a
// corrupt archive, which the record checks reject)
__device__ __noinline__ unsigned long long out_bits(const OutLookup o, uint64_t i) {
    i += o.base;
    const uint64_t b = i >> 10;
    uint64_t lo = o.start[b], hi = o.start[b + 1];
    if (hi > o.k) hi = o.k;
    if (lo > hi) lo = hi;
    if (hi > lo) {   // first probe where evenly spread records would put i (block corners: exact)
        const uint64_t m = lo + (((i & 1023) * (hi - lo)) >> 10);
        const unsigned long long v = o.idx[m * o.stride];
        if (v == i) return o.val[m * o.stride];
        if (v < i) lo = m + 1; else hi = m;
    }
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (o.idx[mid * o.stride] < i) lo = mid + 1; else hi = mid;
    }
    return (lo < o.k && o.idx[lo * o.stride] == i) ? o.val[lo * o.stride] : 0ull;
}
__device__ __forceinline__ long long outlier_int(const OutLookup& o, uint64_t i) {
    return (long long)__longlong_as_double((long long)out_bits(o, i));
}

// segmented (width W lanes) inclusive scan + last-outlier correction
template <int W>
__device__ __forceinline__ long long row_final(int dlt, bool isout, long long vout, long long K,
                                               uint32_t lane) {
    const uint32_t sl = lane & (W - 1);
    int S = dlt;
#pragma unroll
    for (int o = 1; o < W; o <<= 1) {
        int t = __shfl_up_sync(kFull, S, o);
        if (sl >= (uint32_t)o) S += t;
    }
    long long t = isout ? (vout - K - (long long)S) : 0;
    uint32_t m = __ballot_sync(kFull, isout);
    uint32_t segmask = (W == 32) ? kFull : (((1u << W) - 1) << (lane & ~(W - 1)));
    uint32_t mine = m & segmask & (lane == 31 ? kFull : ((2u << lane) - 1));
    int src = mine ? 31 - __clz(mine) : (int)lane;
    long long corr = __shfl_sync(kFull, t, src);
    if (!mine) corr = 0;
    return (long long)S + corr + K;
}

// int32 variant of row_final; the caller guarantees |K| < 3*2^28 and |v| < 2^27
template <int W>
__device__ __forceinline__ int row_final32(int dlt, bool isout, int vout, int K, uint32_t lane) {
    const uint32_t sl = lane & (W - 1);
    int S = dlt;
#pragma unroll
    for (int o = 1; o < W; o <<= 1) {
        const int t = __shfl_up_sync(kFull, S, o);
        if (sl >= (uint32_t)o) S += t;
    }
    const int t = isout ? (vout - K - S) : 0;
    const uint32_t m = __ballot_sync(kFull, isout);
    const uint32_t segmask = (W == 32) ? kFull : (((1u << W) - 1) << (lane & ~(W - 1)));
    const uint32_t mine = m & segmask & (lane == 31 ? kFull : ((2u << lane) - 1));
    const int src = mine ? 31 - __clz(mine) : (int)lane;
    const int corr = __shfl_sync(kFull, t, src);
    return S + (mine ? corr : 0) + K;
}


// ----------------------------------------------------------------------------
// 3D block 8x8x8, one thread per block.  With H = prefix_x(delta),
// G = H + G(row y-1), F = G + F(plane z-1) the Lorenzo inverse costs three
// integer adds per point and needs no communication: F of the previous plane
// (64 values) and G of the previous row (8) live in registers.  An outlier
// fixes F = v and re-derives G and H from it, which is exactly the
// reference's per-outlier box correction applied in raster order
// (dualquant.py:218-226).  A warp covers 32 consecutive blocks along x, so
// every row of 8 codes (16 B) and 8 outputs (32 B) is part of one contiguous
// warp-wide access.  int32 arithmetic with a magnitude guard (|F| < 2^28
// keeps every intermediate exact); a block that trips it is redone in int64.
// ----------------------------------------------------------------------------
// one row of 8 points: x-prefix, then the y and z recurrences; outliers
// (code 0) take their stored value.  Returns false on the magnitude guard.

template <int OUTK>
__device__ __forceinline__ void rq_store8(void* __restrict__ out, uint64_t rb, const int (&F)[8],
                                          double two_eb, int nx, bool vec, const QualArgs& q, QAcc& acc) {
    if (OUTK == 0) {
        float o[8];
#pragma unroll
        for (int x = 0; x < 8; x++) o[x] = __double2float_rn(__dmul_rn((double)F[x], two_eb));
        if (q.orig) {
#pragma unroll
            for (int x = 0; x < 8; x++)
                if (x < nx) acc.add(q, rb + x, (double)o[x]);
        }
        float* op = (float*)out + rb;
        if (vec) {
            *reinterpret_cast<float4*>(op) = make_float4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<float4*>(op + 4) = make_float4(o[4], o[5], o[6], o[7]);
        } else {
#pragma unroll
            for (int x = 0; x < 8; x++)
                if (x < nx) op[x] = o[x];
        }
    } else {
        double* op = (double*)out + rb;
#pragma unroll
        for (int x = 0; x < 8; x++)
            if (vec || x < nx) op[x] = __dmul_rn((double)F[x], two_eb);
        if (q.orig) {
#pragma unroll
            for (int x = 0; x < 8; x++)
                if (x < nx) acc.add(q, rb + x, __dmul_rn((double)F[x], two_eb));
        }
    }
}


// One thread per block (full x-extent, 8-byte aligned rows): F of the previous
// plane lives in shared memory, transposed ([y][x/4][thread] int4) so the
// per-row reads/writes are conflict-free, which keeps registers for the
// prefetched next plane.
constexpr int kRqThreads = 64;

__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// The thread's block rows stream through shared memory: plane z+1's 16
// eight-byte row halves are copied by cp.async while plane z is processed.
// Shared layouts are [slot][thread] so a warp's accesses are contiguous.
template <int OUTK>
__device__ __forceinline__ bool rq3d_block_smem(const uint16_t* __restrict__ codes,
                                                const OutLookup ol,
                                                uint64_t base, uint64_t YX, uint64_t X, int nx, int ny,
                                                int nz, int r, double two_eb, void* __restrict__ out,
                                                int4* __restrict__ fp, uint2* __restrict__ cs, bool vec,
                                                bool vec_out, const QualArgs& q, QAcc& acc) {
    // vec: 8-byte aligned rows whose 16-byte reads stay inside the array
    // (cp.async); otherwise rows are gathered with guarded scalar loads.
    // x >= nx (partial edge block): the row read runs into the next row; those
    // codes are replaced by residual 0 and their values are never stored.
    // Rows past the field (ny < 8) load a clamped row and are never stored.
#pragma unroll
    for (int i = 0; i < 16; i++) fp[i * kRqThreads] = make_int4(0, 0, 0, 0);
    int mx = 0, mn = 0;
    const bool edge = nx < 8;
    auto fetch = [&](int z) {
        const int buf = z & 1;
        for (int y = 0; y < 8; y++) {
            const uint16_t* src = codes + base + (uint64_t)z * YX + (uint64_t)min(y, ny - 1) * X;
            uint2* d0 = cs + ((buf * 8 + y) * 2) * kRqThreads;
            uint2* d1 = d0 + kRqThreads;
            if (vec) {
                cp_async8((uint32_t)__cvta_generic_to_shared(d0), src);
                cp_async8((uint32_t)__cvta_generic_to_shared(d1), src + 4);
            } else {
                uint32_t c[8];
#pragma unroll
                for (int x = 0; x < 8; x++) c[x] = x < nx ? src[x] : (uint32_t)r;
                *d0 = make_uint2(c[0] | (c[1] << 16), c[2] | (c[3] << 16));
                *d1 = make_uint2(c[4] | (c[5] << 16), c[6] | (c[7] << 16));
            }
        }
        cp_async_commit();
    };
    fetch(0);
    // the block corner (first point, zero-padded neighbours) is an outlier in
    // most smooth blocks: its record lookup runs while plane 0's codes arrive
    const long long corner = outlier_int(ol, base);
#pragma unroll 1
    for (int z = 0; z < nz; z++) {
        if (z + 1 < nz) fetch(z + 1);
        else cp_async_commit();   // empty group keeps the wait count uniform
        cp_async_wait1();
        const uint64_t zb = base + (uint64_t)z * YX;
        const uint2* cz = cs + ((z & 1) * 8 * 2) * kRqThreads;
        int Gp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 1
        for (int y = 0; y < 8; y++) {
            const uint2 u0 = cz[(y * 2) * kRqThreads], u1 = cz[(y * 2 + 1) * kRqThreads];
            uint32_t cw[8] = {u0.x & 0xFFFF, u0.x >> 16, u0.y & 0xFFFF, u0.y >> 16,
                              u1.x & 0xFFFF, u1.x >> 16, u1.y & 0xFFFF, u1.y >> 16};
            if (edge) {
#pragma unroll
                for (int x = 0; x < 8; x++) cw[x] = x < nx ? cw[x] : (uint32_t)r;
            }
            const uint64_t rb = zb + (uint64_t)y * X;
            const int4 a = fp[(y * 2) * kRqThreads], b = fp[(y * 2 + 1) * kRqThreads];
            const int F0[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            int F[8], G[8];
            int H = 0;
#pragma unroll
            for (int x = 0; x < 8; x++) {
                H += (int)cw[x] - r;
                G[x] = H + Gp[x];
                F[x] = G[x] + F0[x];
            }
            bool anyz = false;
#pragma unroll
            for (int x = 0; x < 8; x++) anyz |= cw[x] == 0;
            if (anyz) {   // rare: redo the row with its outliers
                H = 0;
#pragma unroll
                for (int x = 0; x < 8; x++) {
                    H += (int)cw[x] - r;
                    G[x] = H + Gp[x];
                    F[x] = G[x] + F0[x];
                    if (cw[x] == 0) {   // outlier: its final value is stored verbatim
                        // rows past the field hold a clamped copy of the last row (never stored)
                        const long long v = (z == 0 && y == 0 && x == 0)
                                                ? corner
                                                : outlier_int(ol, (y < ny ? rb : zb + (uint64_t)(ny - 1) * X) + x);
                        F[x] = (v < (1ll << 28) && v > -(1ll << 28)) ? (int)v : (1 << 29);
                        G[x] = F[x] - F0[x];
                        H = G[x] - Gp[x];
                    }
                }
            }
#pragma unroll
            for (int x = 0; x < 8; x++) {
                Gp[x] = G[x];
                mx = max(mx, F[x]);
                mn = min(mn, F[x]);
            }
            fp[(y * 2) * kRqThreads] = make_int4(F[0], F[1], F[2], F[3]);
            fp[(y * 2 + 1) * kRqThreads] = make_int4(F[4], F[5], F[6], F[7]);
            if (y < ny) rq_store8<OUTK>(out, rb, F, two_eb, nx, OUTK == 0 && !edge && vec_out, q, acc);
        }
    }
    cp_async_wait1();
    return mx < (1 << 28) && mn > -(1 << 28);
}

template <int OUTK>
__global__ void __launch_bounds__(kRqThreads) rq3d_block_kernel(const uint16_t* __restrict__ codes,
                                                         const OutLookup ol,
                                                         uint8_t* __restrict__ blockflag,
                                                         int any_slow, uint64_t Z, uint64_t Y,
                                                         uint64_t X, uint32_t cap, double two_eb,
                                                         void* __restrict__ out, DevStatus* st, QualArgs q) {
    __shared__ int4 s_fp[16 * kRqThreads];
    QAcc acc;
    __shared__ uint2 s_cs[2 * 16 * kRqThreads];
    const int r = (int)(cap >> 1);
    const uint64_t nbx = ceil_div(X, 8), nby = ceil_div(Y, 8), nbz = ceil_div(Z, 8);
    const uint64_t nblk = nbx * nby * nbz;
    const uint64_t YX = Y * X;
    const bool vec_ok = (X & 3) == 0 && ((uintptr_t)codes & 7) == 0;
    const bool vec_out = (X & 3) == 0 && ((uintptr_t)out & 15) == 0;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nblk;
         b += (uint64_t)gridDim.x * blockDim.x) {
        if (any_slow && blockflag[b]) continue;   // the fp64 replay kernel owns it
        const uint64_t bx = b % nbx, t2 = b / nbx, by = t2 % nby, bz = t2 / nby;
        const int nx = (int)umin(8, X - bx * 8), ny = (int)umin(8, Y - by * 8), nz = (int)umin(8, Z - bz * 8);
        const uint64_t base = bz * 8 * YX + by * 8 * X + bx * 8;
        // cp.async rows need 8-byte alignment and the last row's 16-byte read
        // inside the code array
        const bool inside = base + (uint64_t)(nz - 1) * YX + (uint64_t)(ny - 1) * X + 8 <= Z * YX;
        const bool ok = rq3d_block_smem<OUTK>(codes, ol, base, YX, X, nx, ny, nz, r, two_eb, out,
                                              s_fp + threadIdx.x, s_cs + threadIdx.x, vec_ok && inside,
                                              vec_out, q, acc);
        if (!ok) {   // magnitude guard: the fp64 replay kernel redoes the block
            blockflag[b] = 1;
            atomicOr(&st->flags, (unsigned long long)F_OUT_SLOW);
        }
    }
    if (q.orig) qacc_flush(acc, q);
}


template <int OUTK>
__global__ void __launch_bounds__(kThreads) rq2d_kernel(const uint16_t* __restrict__ codes,
                                                        const OutLookup ol,
                                                        const uint8_t* __restrict__ blockflag,
                                                        int any_slow, uint64_t Y, uint64_t X,
                                                        uint32_t cap, double two_eb,
                                                        void* __restrict__ out) {
    const int r = (int)(cap >> 1);
    const uint32_t lane = lane_id();
    const uint64_t nbx = ceil_div(X, 16), nbx2 = ceil_div(nbx, 2), nby = ceil_div(Y, 16);
    const uint64_t ntask = nbx2 * nby;
    for (uint64_t task = blockIdx.x * (uint64_t)kWarpsPerCta + (threadIdx.x >> 5); task < ntask;
         task += (uint64_t)gridDim.x * kWarpsPerCta) {
        const uint64_t bx2 = task % nbx2, by = task / nbx2;
        const uint64_t x = bx2 * 32 + lane, y0 = by * 16;
        const bool xin = x < X;
        bool skip = false;
        if (any_slow && xin) skip = blockflag[by * nbx + (x >> 4)] != 0;
        const int ny = (int)umin(16, Y - y0);
        long long prev = 0;
        for (int y = 0; y < ny; y++) {
            const uint64_t i = (y0 + y) * X + x;
            uint32_t code = xin ? codes[i] : (uint32_t)r;
            const bool isout = xin && code == 0;
            const int dlt = isout ? 0 : (int)code - r;
            const long long vout = isout ? outlier_int(ol, i) : 0;
            const long long fin = row_final<16>(dlt, isout, vout, prev, lane);
            prev = fin;
            if (xin && !skip) store_out<OUTK>(out, i, fin, two_eb);
        }
    }
}

// 2D block 16x16, row pitch a multiple of 4: a task is 16 rows x 128 columns
// (8 blocks), lane l holds columns 4l..4l+3 (uint2 code loads, all 16 rows in
// flight; float4 stores), a block spans 4 lanes.  Row recurrence
// F(y, x) = F(y-1, x) + S_y(x), S_y = x-prefix of the residuals restarted at an
// outlier p with S_y(p) = v - F(y-1, p) -- the reference's per-outlier box
// correction (dualquant.py:218-226) in raster order -- as a reset scan over
// the block's 4 lanes.  int32 unless an outlier value of the task reaches
// 2^29 (then |F| < 2^29 + 256 r keeps every result exact; wrapped partial sums
// cancel).
template <typename V, int OUTK>
__device__ __forceinline__ void rq2d_vec_rows(const uint2 (&cw)[16], const OutLookup ol,
                                              uint64_t X, uint64_t y0, int ny, uint64_t x0, bool xin, bool store,
                                              int r, uint32_t lane, double two_eb, void* __restrict__ out,
                                              const QualArgs& q, QAcc& acc) {
    V K[4] = {0, 0, 0, 0};
    const uint32_t sl = lane & 3;
    const uint32_t below = ((1u << sl) - 1u) << (lane & ~3u);
#pragma unroll
    for (int y = 0; y < 16; y++) {
        const bool row = xin && y < ny;
        const uint64_t i0 = (y0 + y) * X + x0;
        const uint32_t c[4] = {cw[y].x & 0xFFFFu, cw[y].x >> 16, cw[y].y & 0xFFFFu, cw[y].y >> 16};
        V loc[4], t = 0;
        bool f = false;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (c[k] == 0) {
                t = (V)__longlong_as_double((long long)out_bits(ol, i0 + k)) - K[k];
                f = true;
            } else {
                t += (V)((int)c[k] - r);
            }
            loc[k] = t;
        }
        V P = t;
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
            const V yv = __shfl_up_sync(kFull, P, o);
            if (sl >= (uint32_t)o) P += yv;
        }
        const V E = P - t;
        const uint32_t m = __ballot_sync(kFull, f) & below;
        const int src = m ? 31 - __clz(m) : (int)(lane & ~3u);
        const V carry = E - __shfl_sync(kFull, E, src);
        bool hit = false;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            hit |= c[k] == 0;
            K[k] += loc[k] + (hit ? (V)0 : carry);
        }
        if (row && store) {
            if (OUTK == 0) {
                float4 o4;
                o4.x = __double2float_rn(__dmul_rn((double)K[0], two_eb));
                o4.y = __double2float_rn(__dmul_rn((double)K[1], two_eb));
                o4.z = __double2float_rn(__dmul_rn((double)K[2], two_eb));
                o4.w = __double2float_rn(__dmul_rn((double)K[3], two_eb));
                __stcs(reinterpret_cast<float4*>((float*)out + i0), o4);
                if (q.orig) {
                    acc.add(q, i0, (double)o4.x);
                    acc.add(q, i0 + 1, (double)o4.y);
                    acc.add(q, i0 + 2, (double)o4.z);
                    acc.add(q, i0 + 3, (double)o4.w);
                }
            } else {
#pragma unroll
                for (int k = 0; k < 4; k++) ((double*)out)[i0 + k] = __dmul_rn((double)K[k], two_eb);
                if (q.orig) {
#pragma unroll
                    for (int k = 0; k < 4; k++) acc.add(q, i0 + k, __dmul_rn((double)K[k], two_eb));
                }
            }
        }
    }
}

template <int OUTK>
__global__ void __launch_bounds__(kThreads, 3) rq2d_vec_kernel(const uint16_t* __restrict__ codes,
                                                            const OutLookup ol,
                                                            const uint8_t* __restrict__ blockflag,
                                                            int any_slow, uint64_t Y, uint64_t X,
                                                            uint32_t cap, double two_eb,
                                                            void* __restrict__ out, QualArgs q) {
    const int r = (int)(cap >> 1);
    const uint32_t lane = lane_id();
    QAcc acc;
    const uint64_t nbx = ceil_div(X, 16), ntx = ceil_div(X, 128), nty = ceil_div(Y, 16);
    const uint64_t ntask = ntx * nty;
    const bool big = *ol.big != 0;
    for (uint64_t task = blockIdx.x * (uint64_t)kWarpsPerCta + (threadIdx.x >> 5); task < ntask;
         task += (uint64_t)gridDim.x * kWarpsPerCta) {
        const uint64_t tx = task % ntx, ty = task / ntx;
        const uint64_t x0 = tx * 128 + lane * 4, y0 = ty * 16;
        const bool xin = x0 < X;
        const int ny = (int)umin(16, Y - y0);
        uint2 cw[16];
#pragma unroll
        for (int y = 0; y < 16; y++) {
            // rows past the field read as residual 0 (code r) and are never stored
            cw[y] = make_uint2((uint32_t)r | ((uint32_t)r << 16), (uint32_t)r | ((uint32_t)r << 16));
            if (xin && y < ny) cw[y] = __ldcs(reinterpret_cast<const uint2*>(codes + (y0 + y) * X + x0));
        }
        const bool store = !(any_slow && xin && blockflag[ty * nbx + (x0 >> 4)]);
        if (big)   // some outlier value >= 2^29 (task_bounds_kernel): int64 rows
            rq2d_vec_rows<long long, OUTK>(cw, ol, X, y0, ny, x0, xin, store, r, lane, two_eb, out, q, acc);
        else
            rq2d_vec_rows<int, OUTK>(cw, ol, X, y0, ny, x0, xin, store, r, lane, two_eb, out, q, acc);
    }
    if (q.orig) qacc_flush(acc, q);
}

template <int OUTK>
__global__ void __launch_bounds__(kThreads) rq1d_kernel(const uint16_t* __restrict__ codes,
                                                        const OutLookup ol,
                                                        const uint8_t* __restrict__ blockflag,
                                                        int any_slow, uint64_t X, uint32_t cap,
                                                        double two_eb, void* __restrict__ out) {
    const int r = (int)(cap >> 1);
    const uint32_t lane = lane_id();
    const uint64_t nb = ceil_div(X, 32);
    for (uint64_t b = blockIdx.x * (uint64_t)kWarpsPerCta + (threadIdx.x >> 5); b < nb;
         b += (uint64_t)gridDim.x * kWarpsPerCta) {
        if (any_slow && blockflag[b]) continue;
        const uint64_t i = b * 32 + lane;
        const bool in = i < X;
        uint32_t code = in ? codes[i] : (uint32_t)r;
        const bool isout = in && code == 0;
        const int dlt = isout ? 0 : (int)code - r;
        const long long vout = isout ? outlier_int(ol, i) : 0;
        const long long fin = row_final<32>(dlt, isout, vout, 0, lane);
        if (in) store_out<OUTK>(out, i, fin, two_eb);
    }
}

// 1D block 32, whole 1024-point tasks: lane l holds points 4l..4l+3 of each of
// the task's 8 rows of 128 (uint2 code loads, all 8 in flight; float4
// stores), a block spans 8 lanes.  Per lane: T = sum of the residuals after
// its last outlier (reset to the outlier's value v there).  Inclusive scan P
// of T over the block's lanes; a lane's carry-in is P(l-1) - P(s-1), s the
// last lane left of it (in the block) holding an outlier -- the reference's
// per-outlier box correction (dualquant.py:218-226) as a reset scan.  The
// scan runs in int32: partial sums wrap, but the carry and every final value
// are exact whenever |v| < 2^30 (then |final| < 2^30 + 32 r < 2^31); a task
// with a larger outlier value takes the int64 instantiation.
// reset scan of one row given the outlier values of its zero codes (vout[k]);
// positions >= nvalid are not stored
template <typename V, int OUTK>
__device__ __forceinline__ void rq1d_rec_row(const uint32_t (&c)[4], const V (&vout)[4], uint64_t i0,
                                             uint32_t nvalid, int r, uint32_t lane, double two_eb,
                                             void* __restrict__ out, bool store, const QualArgs& q, QAcc& acc) {
    V fin[4];
    V t = 0;
    bool f = false;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        t = c[k] == 0 ? vout[k] : t + (V)((int)c[k] - r);
        f |= c[k] == 0;
        fin[k] = t;
    }
    const uint32_t sl = lane & 7;
    V P = t;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        const V y = __shfl_up_sync(kFull, P, o);
        if (sl >= (uint32_t)o) P += y;
    }
    const V E = P - t;
    const uint32_t m = __ballot_sync(kFull, f) & (((1u << sl) - 1u) << (lane & ~7u));
    const int s = m ? 31 - __clz(m) : (int)(lane & ~7u);
    const V carry = E - __shfl_sync(kFull, E, s);
    bool hit = false;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        hit |= c[k] == 0;
        if (!hit) fin[k] += carry;
    }
    if (!store) return;
    if (OUTK == 0 && nvalid >= 4) {
        float4 o4;
        o4.x = __double2float_rn(__dmul_rn((double)fin[0], two_eb));
        o4.y = __double2float_rn(__dmul_rn((double)fin[1], two_eb));
        o4.z = __double2float_rn(__dmul_rn((double)fin[2], two_eb));
        o4.w = __double2float_rn(__dmul_rn((double)fin[3], two_eb));
        __stcs(reinterpret_cast<float4*>((float*)out + i0), o4);
        if (q.orig) {
            acc.add(q, i0, (double)o4.x);
            acc.add(q, i0 + 1, (double)o4.y);
            acc.add(q, i0 + 2, (double)o4.z);
            acc.add(q, i0 + 3, (double)o4.w);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if ((uint32_t)k < nvalid) {
                store_out<OUTK>(out, i0 + k, (long long)fin[k], two_eb);
                if (q.orig) {
                    const double v = __dmul_rn((double)fin[k], two_eb);
                    acc.add(q, i0 + k, OUTK == 0 ? (double)__double2float_rn(v) : v);
                }
            }
        }
    }
}

// start[t] = first record with index >= 1024 t (lower bound; t <= ntask)
// first record of every 1024-point bucket (lower bound of t * 1024 over the
// record indices idx[j * stride]; bounded whatever the order of a corrupt set).
// (A galloping search from the evenly-spread guess measured slower: the 3D
// block-corner outliers cluster in every 64th row of buckets.)
__global__ void task_bounds_kernel(const unsigned long long* __restrict__ idx,
                                   const unsigned long long* __restrict__ val, uint32_t stride, uint64_t k,
                                   uint64_t ntask, unsigned long long* __restrict__ start) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t <= ntask;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = t * 1024ull;
        uint64_t lo = 0, hi = k;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (idx[mid * stride] < key) lo = mid + 1; else hi = mid;
        }
        start[t] = lo;
    }
    // start[ntask + 1]: some record's value is at least 2^29 in magnitude (or NaN):
    // the int32 2D reconstruct is not exact for it (zeroed by the launcher)
    bool big = false;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < k; j += (uint64_t)gridDim.x * blockDim.x)
        big |= !(fabs(__longlong_as_double((long long)val[j * stride])) < 536870912.0);
    if (__any_sync(kFull, big) && lane_id() == 0) atomicOr(&start[ntask + 1], 1ull);
}

// the 8 rows of a task; zero codes take the value of the task record of the
// same rank (task-relative ranks, first kVals values staged in `vals`)
constexpr uint32_t kVals = 64;
template <bool FULL, typename V, int OUTK>
__device__ __forceinline__ void rq1d_rec_rows(const uint2 (&cw)[8], const double* vals,
                                              const unsigned long long* __restrict__ trec, uint32_t m,
                                              uint64_t t0, uint64_t n, const uint8_t* __restrict__ blockflag,
                                              bool any_slow, int r, uint32_t lane, double two_eb,
                                              void* __restrict__ out, const QualArgs& qa, QAcc& acc) {
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t base = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const uint64_t i0 = t0 + j * 128 + lane * 4;
        const uint32_t nvalid = FULL ? 4u : (i0 >= n ? 0u : (uint32_t)umin(4, n - i0));
        const uint32_t c[4] = {cw[j].x & 0xFFFFu, cw[j].x >> 16, cw[j].y & 0xFFFFu, cw[j].y >> 16};
        bool z[4];
#pragma unroll
        for (int q = 0; q < 4; q++) z[q] = c[q] == 0 && (FULL || (uint32_t)q < nvalid);
        const bool store = (FULL || nvalid) && !(any_slow && blockflag[i0 >> 5]);
        const uint32_t b0 = __ballot_sync(kFull, z[0]), b1 = __ballot_sync(kFull, z[1]),
                       b2 = __ballot_sync(kFull, z[2]), b3 = __ballot_sync(kFull, z[3]);
        V v4[4] = {0, 0, 0, 0};
        if (b0 | b1 | b2 | b3) {
            uint32_t rk = base + __popc(b0 & lt) + __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                if (z[q]) {
                    const double v = rk < kVals ? (rk < m ? vals[rk] : 0.0)
                                                : (rk < m ? __longlong_as_double((long long)trec[2 * rk + 1]) : 0.0);
                    v4[q] = (V)v;
                    rk++;
                }
            }
            base += __popc(b0) + __popc(b1) + __popc(b2) + __popc(b3);
        }
        rq1d_rec_row<V, OUTK>(c, v4, i0, FULL ? 4u : nvalid, r, lane, two_eb, out, store, qa, acc);
    }
}

// 1D block 32 from the archive's sorted outlier records (no dense scatter):
// task t = points [1024 t, 1024 t + 1024) owns records [start[t], start[t+1]).
// Each record's code is fetched from the lanes holding the task's codes
// (codes[idx] == 0, dualquant.py:290-291); a zero code's value is the record
// of the same rank among the task's zero codes (equal sets once the count
// check of dualquant.py:292-294 passes, which the host makes after this).
template <int OUTK>
__global__ void __launch_bounds__(kThreads, 4) rq1d_rec_kernel(const uint16_t* __restrict__ codes,
                                                            const unsigned long long* __restrict__ rec,
                                                            const unsigned long long* __restrict__ start,
                                                            uint64_t k, const uint8_t* __restrict__ blockflag,
                                                            uint64_t n, uint32_t cap, double two_eb,
                                                            void* __restrict__ out, DevStatus* st, QualArgs qa) {
    __shared__ double s_vals[kWarpsPerCta][kVals];
    QAcc acc;
    const int r = (int)(cap >> 1);
    const uint32_t lane = lane_id();
    double* const vals = s_vals[threadIdx.x >> 5];
    const uint64_t ntask = ceil_div(n, 1024);
    const bool any_slow = (st->flags & F_OUT_SLOW) != 0;
    bool nz = false;
    for (uint64_t task = blockIdx.x * (uint64_t)kWarpsPerCta + (threadIdx.x >> 5); task < ntask;
         task += (uint64_t)gridDim.x * kWarpsPerCta) {
        const uint64_t t0 = task * 1024;
        const bool full = t0 + 1024 <= n;
        uint2 cw[8];
        if (full) {
            const uint2* src = reinterpret_cast<const uint2*>(codes + t0) + lane;
#pragma unroll
            for (int j = 0; j < 8; j++) cw[j] = __ldcs(src + 32 * j);
        } else {
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const uint64_t i0 = t0 + j * 128 + lane * 4;
                uint32_t h[4];
#pragma unroll
                for (int q = 0; q < 4; q++) h[q] = i0 + q < n ? codes[i0 + q] : (uint32_t)r;
                cw[j] = make_uint2(h[0] | (h[1] << 16), h[2] | (h[3] << 16));
            }
        }
        uint64_t s0 = start[task], s1 = start[task + 1];
        s0 = s0 < k ? s0 : k;
        s1 = s1 < s0 ? s0 : (s1 < k ? s1 : k);
        // the task's records: code at each index must be 0; values beyond
        // 2^30 in magnitude send the task to int64
        bool big = false;
        for (uint64_t b = s0; b < s1; b += 32) {
            const uint64_t q = b + lane;
            const bool has = q < s1;
            const unsigned long long idx = has ? rec[2 * q] : t0;
            const double v = has ? __longlong_as_double((long long)rec[2 * q + 1]) : 0.0;
            const uint64_t p = idx - t0;
            const uint32_t row = (uint32_t)(p >> 7) & 7u, src = (uint32_t)(p >> 2) & 31u, kk = (uint32_t)p & 3u;
            uint32_t word = 0;
#pragma unroll
            for (int jj = 0; jj < 8; jj++) {
                const uint32_t wx = __shfl_sync(kFull, cw[jj].x, src), wy = __shfl_sync(kFull, cw[jj].y, src);
                if ((uint32_t)jj == row) word = kk < 2 ? wx : wy;
            }
            const uint32_t code = (word >> (16 * (kk & 1))) & 0xFFFFu;
            nz |= has && p < 1024 && code != 0;
            big |= has && !(fabs(v) < 1073741824.0);
            if (has && q - s0 < kVals) vals[q - s0] = v;
        }
        __syncwarp();
        const bool wide = __any_sync(kFull, big);
        const uint32_t m = (uint32_t)(s1 - s0);   // records of the task (< 2^31: <= 1024 if consistent)
        if (full) {
            if (wide) rq1d_rec_rows<true, long long, OUTK>(cw, vals, rec + 2 * s0, m, t0, n, blockflag, any_slow, r, lane, two_eb, out, qa, acc);
            else rq1d_rec_rows<true, int, OUTK>(cw, vals, rec + 2 * s0, m, t0, n, blockflag, any_slow, r, lane, two_eb, out, qa, acc);
        } else {
            if (wide) rq1d_rec_rows<false, long long, OUTK>(cw, vals, rec + 2 * s0, m, t0, n, blockflag, any_slow, r, lane, two_eb, out, qa, acc);
            else rq1d_rec_rows<false, int, OUTK>(cw, vals, rec + 2 * s0, m, t0, n, blockflag, any_slow, r, lane, two_eb, out, qa, acc);
        }
        __syncwarp();
    }
    if (__any_sync(kFull, nz) && lane == 0) atomicOr(&st->flags, (unsigned long long)F_OUT_NONZERO);
    if (qa.orig) qacc_flush(acc, qa);
}

template <typename V, int OUTK>
__device__ __forceinline__ void rq1d_vec_row(uint2 cw, const OutLookup ol,
                                             uint64_t i0, int r, uint32_t lane, double two_eb,
                                             void* __restrict__ out, bool store) {
    const uint32_t c[4] = {cw.x & 0xFFFFu, cw.x >> 16, cw.y & 0xFFFFu, cw.y >> 16};
    V fin[4];
    V t = 0;
    bool f = false;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        if (c[k] == 0) {
            t = (V)__longlong_as_double((long long)out_bits(ol, i0 + k));
            f = true;
        } else {
            t += (V)((int)c[k] - r);
        }
        fin[k] = t;   // local value (carry added below)
    }
    // inclusive scan of t over the block's 8 lanes
    const uint32_t sl = lane & 7;
    V P = t;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        const V y = __shfl_up_sync(kFull, P, o);
        if (sl >= (uint32_t)o) P += y;
    }
    const V E = P - t;   // exclusive
    const uint32_t m = __ballot_sync(kFull, f) & (((1u << sl) - 1u) << (lane & ~7u));
    const int s = m ? 31 - __clz(m) : (int)(lane & ~7u);
    const V Es = __shfl_sync(kFull, E, s);
    const V carry = E - Es;
    bool hit = false;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        hit |= c[k] == 0;
        if (!hit) fin[k] += carry;
    }
    if (!store) return;
    if (OUTK == 0) {
        float4 o4;
        o4.x = __double2float_rn(__dmul_rn((double)fin[0], two_eb));
        o4.y = __double2float_rn(__dmul_rn((double)fin[1], two_eb));
        o4.z = __double2float_rn(__dmul_rn((double)fin[2], two_eb));
        o4.w = __double2float_rn(__dmul_rn((double)fin[3], two_eb));
        __stcs(reinterpret_cast<float4*>((float*)out + i0), o4);
    } else {
        double* o = (double*)out + i0;
#pragma unroll
        for (int k = 0; k < 4; k++) o[k] = __dmul_rn((double)fin[k], two_eb);
    }
}

template <int OUTK>
__global__ void __launch_bounds__(kThreads) rq1d_vec_kernel(const uint16_t* __restrict__ codes,
                                                            const OutLookup ol,
                                                            const uint8_t* __restrict__ blockflag,
                                                            int any_slow, uint64_t ntask, uint32_t cap,
                                                            double two_eb, void* __restrict__ out) {
    const int r = (int)(cap >> 1);
    const uint32_t lane = lane_id();
    for (uint64_t task = blockIdx.x * (uint64_t)kWarpsPerCta + (threadIdx.x >> 5); task < ntask;
         task += (uint64_t)gridDim.x * kWarpsPerCta) {
        const uint64_t t0 = task * 1024;
        const uint2* src = reinterpret_cast<const uint2*>(codes + t0) + lane;
        uint2 cw[8];
#pragma unroll
        for (int j = 0; j < 8; j++) cw[j] = __ldcs(src + 32 * j);
        // an outlier value at or beyond 2^30 in magnitude sends the task to int64
        bool big = false;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint32_t z = __vcmpeq2(cw[j].x, 0u) | __vcmpeq2(cw[j].y, 0u);
            if (z) {
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const uint32_t cc = k < 2 ? (cw[j].x >> (16 * k)) & 0xFFFFu : (cw[j].y >> (16 * (k - 2))) & 0xFFFFu;
                    if (cc == 0) {
                        const double v = __longlong_as_double((long long)out_bits(ol, t0 + j * 128 + lane * 4 + k));
                        big |= !(fabs(v) < 1073741824.0);
                    }
                }
            }
        }
        const bool wide = __any_sync(kFull, big);
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint64_t i0 = t0 + j * 128 + lane * 4;
            const bool store = !(any_slow && blockflag[i0 >> 5]);
            if (wide) rq1d_vec_row<long long, OUTK>(cw[j], ol, i0, r, lane, two_eb, out, store);
            else rq1d_vec_row<int, OUTK>(cw[j], ol, i0, r, lane, two_eb, out, store);
        }
    }
}

// Reference-order fp64 reconstruction, one thread per block (generic shapes
// and flagged blocks).  `work` is an fp64 scratch array indexed like the field.
template <int OUTK>
__global__ void rq_generic_kernel(const uint16_t* __restrict__ codes,
                                  const OutLookup ol,
                                  const uint8_t* __restrict__ blockflag, int only_flagged, Geo g,
                                  uint32_t cap, double two_eb, double* __restrict__ work,
                                  void* __restrict__ out, const DevStatus* st, uint64_t slot_pts) {
    if (only_flagged && !(st->flags & F_OUT_SLOW)) return;
    const double r = (double)(cap >> 1);
    const uint64_t nblocks = g.nblk[0] * g.nblk[1] * g.nblk[2];
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nblocks;
         b += (uint64_t)gridDim.x * blockDim.x) {
        if (only_flagged && !blockflag[b]) continue;
        uint64_t bc[3] = {0, 0, 0}, rem = b;
        for (int a = g.nd - 1; a >= 0; a--) { bc[a] = rem % g.nblk[a]; rem /= g.nblk[a]; }
        uint64_t o[3] = {0, 0, 0}, e[3] = {1, 1, 1};
        for (int a = 0; a < g.nd; a++) {
            o[a] = bc[a] * g.block[a];
            e[a] = umin(g.block[a], g.dims[a] - o[a]);
        }
        uint64_t st0 = g.nd > 0 ? g.stride[0] : 1, st1 = g.nd > 1 ? g.stride[1] : 1,
                 st2 = g.nd > 2 ? g.stride[2] : 1;
        uint64_t base = o[0] * st0 + (g.nd > 1 ? o[1] * st1 : 0) + (g.nd > 2 ? o[2] * st2 : 0);
        auto gat = [&](uint64_t a, uint64_t bb, uint64_t c) { return base + a * st0 + bb * st1 + c * st2; };
        // work: the whole-field array (all blocks), or this thread's block-sized
        // slot (slot_pts >= the block's points) when only flagged blocks are replayed
        const uint64_t wbase = only_flagged ? (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * slot_pts : 0;
        auto at = [&](uint64_t a, uint64_t bb, uint64_t c) {
            return only_flagged ? wbase + (a * e[1] + bb) * e[2] + c : gat(a, bb, c);
        };
        // residuals
        for (uint64_t a = 0; a < e[0]; a++)
            for (uint64_t bb = 0; bb < e[1]; bb++)
                for (uint64_t c = 0; c < e[2]; c++) {
                    const uint32_t code = codes[gat(a, bb, c)];
                    work[at(a, bb, c)] = code == 0 ? 0.0 : __dsub_rn((double)code, r);
                }
        // cumsum along block axis 0, then 1, then 2 (dualquant.py:215-217)
        for (uint64_t bb = 0; bb < e[1]; bb++)
            for (uint64_t c = 0; c < e[2]; c++)
                for (uint64_t a = 1; a < e[0]; a++)
                    work[at(a, bb, c)] = __dadd_rn(work[at(a, bb, c)], work[at(a - 1, bb, c)]);
        if (g.nd > 1)
            for (uint64_t a = 0; a < e[0]; a++)
                for (uint64_t c = 0; c < e[2]; c++)
                    for (uint64_t bb = 1; bb < e[1]; bb++)
                        work[at(a, bb, c)] = __dadd_rn(work[at(a, bb, c)], work[at(a, bb - 1, c)]);
        if (g.nd > 2)
            for (uint64_t a = 0; a < e[0]; a++)
                for (uint64_t bb = 0; bb < e[1]; bb++)
                    for (uint64_t c = 1; c < e[2]; c++)
                        work[at(a, bb, c)] = __dadd_rn(work[at(a, bb, c)], work[at(a, bb, c - 1)]);
        // outliers in raster order: acc[box] += v - acc[p]   (dualquant.py:218-226)
        for (uint64_t a = 0; a < e[0]; a++)
            for (uint64_t bb = 0; bb < e[1]; bb++)
                for (uint64_t c = 0; c < e[2]; c++) {
                    const uint64_t gi = gat(a, bb, c);
                    if (codes[gi] != 0) continue;
                    double v = __longlong_as_double((long long)out_bits(ol, gi));
                    double d = __dsub_rn(v, work[at(a, bb, c)]);
                    for (uint64_t a2 = a; a2 < e[0]; a2++)
                        for (uint64_t b2 = bb; b2 < e[1]; b2++)
                            for (uint64_t c2 = c; c2 < e[2]; c2++) {
                                uint64_t j = at(a2, b2, c2);
                                work[j] = __dadd_rn(work[j], d);
                            }
                }
        for (uint64_t a = 0; a < e[0]; a++)
            for (uint64_t bb = 0; bb < e[1]; bb++)
                for (uint64_t c = 0; c < e[2]; c++) {
                    const uint64_t gi = gat(a, bb, c);
                    double v = __dmul_rn(work[at(a, bb, c)], two_eb);
                    if (OUTK == 0) ((float*)out)[gi] = __double2float_rn(v);
                    else ((double*)out)[gi] = v;
                }
    }
}

// Generic block shapes, one thread per block (row f4; the fast shapes have
// their own kernels): the block is walked in raster order with the same
// integer recurrence as rq3d_block_kernel -- H = prefix_x(delta), G = H + G of
// row y-1, F = G + F of plane z-1, an outlier fixing F = v and re-deriving G,
// H (the reference's box corrections in raster order, dualquant.py:218-226).
// G of the previous row and F of the previous plane sit in the thread's
// shared-memory slots ([slot][thread]); each is read and overwritten in
// place.  int32 with the fast kernels' magnitude guard: a block that trips it
// (or holds a non-integer outlier value, flagged by the scatter) is replayed
// in the reference's fp64 order by rq_generic_kernel.
constexpr uint32_t kBlkMaxSlots = 1024;   // per-thread int32 slots (4 KB)

__host__ __device__ __forceinline__ uint32_t blk_slots(int nd, const uint32_t* block) {
    const uint32_t bx = block[nd - 1], by = nd >= 2 ? block[nd - 2] : 1;
    return (nd == 3 ? bx * by : 0) + (nd >= 2 ? bx : 0);
}

template <int OUTK, int ND>
__global__ void __launch_bounds__(64) rq_blocks_kernel(const uint16_t* __restrict__ codes,
                                                       const OutLookup ol,
                                                       uint8_t* __restrict__ blockflag, Geo g, uint32_t cap,
                                                       double two_eb, void* __restrict__ out, DevStatus* st) {
    extern __shared__ __align__(16) int blk_smem[];
    const uint32_t T = blockDim.x, tid = threadIdx.x;
    const int nd = ND ? ND : g.nd;   // ND 0: runtime (1D measured faster that way)
    const uint32_t bx = g.block[nd - 1], by = nd >= 2 ? g.block[nd - 2] : 1, bz = nd == 3 ? g.block[0] : 1;
    int* P = blk_smem + tid;                                      // [by][bx]: F of plane z-1 (3D)
    int* Gs = P + (size_t)(nd == 3 ? bx * by : 0) * T;            // [bx]: G of row y-1 (2D, 3D)
    const uint64_t nbx = g.nblk[nd - 1], nby = nd >= 2 ? g.nblk[nd - 2] : 1;
    const uint64_t nblocks = g.nblk[0] * g.nblk[1] * g.nblk[2];
    const uint64_t sy = nd >= 2 ? g.stride[nd - 2] : 0, sz = nd == 3 ? g.stride[0] : 0;
    const uint64_t X = g.dims[nd - 1], Y = nd >= 2 ? g.dims[nd - 2] : 1, Z = nd == 3 ? g.dims[0] : 1;
    const int r = (int)(cap >> 1);
    for (uint64_t b = blockIdx.x * (uint64_t)T + tid; b < nblocks; b += (uint64_t)gridDim.x * T) {
        if (blockflag[b]) continue;   // non-integer outlier value: the fp64 replay owns it
        const uint64_t cx = b % nbx, t2 = b / nbx, cy = t2 % nby, cz = t2 / nby;
        const uint32_t nx = (uint32_t)umin(bx, X - cx * bx), ny = (uint32_t)umin(by, Y - cy * by),
                       nz = (uint32_t)umin(bz, Z - cz * bz);
        const uint64_t base = cz * bz * sz + cy * by * sy + cx * bx;
        int mx = 0, mn = 0;
        for (uint32_t z = 0; z < nz; z++) {
            for (uint32_t y = 0; y < ny; y++) {
                const uint64_t rb = base + z * sz + y * sy;
                int H = 0;
                for (uint32_t x = 0; x < nx; x++) {
                    const uint32_t code = codes[rb + x];
                    const int Gp = (nd >= 2 && y > 0) ? Gs[(size_t)x * T] : 0;
                    int* pf = P + (size_t)(y * bx + x) * T;
                    const int F0 = (nd == 3 && z > 0) ? *pf : 0;
                    int G, F;
                    if (code != 0) {
                        H += (int)code - r;
                        G = H + Gp;
                        F = G + F0;
                    } else {   // outlier: its final value is stored verbatim
                        const long long v = outlier_int(ol, rb + x);
                        F = (v < (1ll << 28) && v > -(1ll << 28)) ? (int)v : (1 << 29);
                        G = F - F0;
                        H = G - Gp;
                    }
                    mx = max(mx, F);
                    mn = min(mn, F);
                    if (nd == 3) *pf = F;
                    if (nd >= 2) Gs[(size_t)x * T] = G;
                    store_out<OUTK>(out, rb + x, F, two_eb);
                }
            }
        }
        if (!(mx < (1 << 28) && mn > -(1 << 28))) {   // magnitude guard: the fp64 replay redoes the block
            blockflag[b] = 1;
            atomicOr(&st->flags, (unsigned long long)F_OUT_SLOW);
        }
    }
}

constexpr int kRowPf = 8;   // row-kernel iterations whose code loads are issued together

// one task of rq1d_seg_kernel with F in V (int32 when every value fits, else int64)
template <typename V, int OUTK>
__device__ __forceinline__ void rq1d_seg_task(const uint16_t* __restrict__ codes, const OutLookup& ol,
                                              uint64_t t0, uint64_t t1, uint32_t bx, int r, uint32_t lane,
                                              unsigned upto, double two_eb, void* __restrict__ out) {
    const uint32_t step = 32 % bx;
    V carry = 0;
    uint32_t pos = lane % bx;
    for (uint64_t g0 = t0; g0 < t1; g0 += 32 * kRowPf) {
        uint32_t cc[kRowPf];   // the group's codes, loaded together
#pragma unroll
        for (int k = 0; k < kRowPf; k++) {
            const uint64_t i = g0 + 32 * k + lane;
            cc[k] = i < t1 ? (uint32_t)codes[i] : (uint32_t)r;
        }
#pragma unroll
        for (int k = 0; k < kRowPf; k++) {
            const uint64_t i0 = g0 + 32 * k;
            if (i0 >= t1) break;
            const uint64_t i = i0 + lane;
            const bool in = i < t1;
            const uint32_t code = cc[k];
            bool reset = pos == 0;
            V b = (V)((int)code - r);
            if (code == 0) {
                reset = true;
                b = (V)(long long)__longlong_as_double((long long)out_bits(ol, i));
            }
            V S = b;   // inclusive prefix sum, restarted at the last reset lane at or left of this one
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const V u = __shfl_up_sync(kFull, S, o);
                if (lane >= (uint32_t)o) S += u;
            }
            const unsigned m = __ballot_sync(kFull, reset) & upto;
            const int L = 31 - __clz((int)m);
            const V Sx = __shfl_sync(kFull, S - b, L < 0 ? 0 : L);
            const V F = m ? S - Sx : carry + S;
            if (in) store_out<OUTK>(out, i, (long long)F, two_eb);
            carry = __shfl_sync(kFull, F, 31);
            pos += step;
            if (pos >= bx) pos -= bx;
        }
    }
}

// 1D generic block length bx >= 32: a warp per task of whole blocks (>= 1024
// points), lane = point, 32 points per step.  The reconstruct is the linear
// recurrence F_i = F_{i-1} + delta_i restarted at a block start (F = delta)
// and at an outlier (F = v): a warp prefix sum minus its value just before
// the last restart lane at or left of each lane (the previous step's F as
// carry when there is none).  int32 when every outlier value is below 2^29
// (task_bounds_kernel's flag) and bx * r < 2^29 (then |F| < 2^30 throughout),
// else int64.  Blocks whose outlier values are not integers below 2^40 are
// flagged by the scatter and rewritten afterwards by the fp64 replay.
template <int OUTK>
__global__ void __launch_bounds__(256) rq1d_seg_kernel(const uint16_t* __restrict__ codes, const OutLookup ol,
                                                       uint64_t n, uint32_t bx, uint64_t task, uint32_t cap,
                                                       double two_eb, void* __restrict__ out, int narrow_ok) {
    const uint32_t lane = lane_id();
    const int r = (int)(cap >> 1);
    const uint64_t ntask = ceil_div(n, task);
    const unsigned upto = (2u << lane) - 1u;   // lanes 0..lane (lane 31: all)
    const bool narrow = narrow_ok && *ol.big == 0;
    for (uint64_t t = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); t < ntask;
         t += (uint64_t)gridDim.x * (blockDim.x >> 5)) {
        const uint64_t t0 = t * task, t1 = umin(t0 + task, n);
        if (narrow) rq1d_seg_task<int, OUTK>(codes, ol, t0, t1, bx, r, lane, upto, two_eb, out);
        else rq1d_seg_task<long long, OUTK>(codes, ol, t0, t1, bx, r, lane, upto, two_eb, out);
    }
}

// 2D / 3D generic block shapes: a warp per strip of block columns -- 32 / bx
// whole blocks side by side when bx <= 32 (ONE), one block of `steps` 32-lane
// segments otherwise -- over nyb consecutive block rows; lane = column.  Rows
// go sequentially; inside a row H (the x prefix of the Lorenzo deltas) is a
// warp prefix sum restarted at the last reset lane at or left of each lane
// (block start, or an outlier whose H is v - F0 - Gp), so G = H + Gp (G of
// row y-1 in this plane) and F = G + F0 (F of the row in plane z-1).  Gp and
// F0 are lane-private shared-memory slots.  int32 modular arithmetic with the
// rq_blocks_kernel magnitude guard: the sequentially first |F| >= 2^28 is
// computed exactly, so a block that trips it is flagged and rewritten by the
// fp64 replay.
template <int OUTK, bool ONE, int ND>
__global__ void __launch_bounds__(256, 4) rq_rows_kernel(const uint16_t* __restrict__ codes, const OutLookup ol,
                                                      uint8_t* __restrict__ blockflag, Geo g, uint32_t W,
                                                      uint32_t steps, uint32_t nyb, uint32_t cap, double two_eb,
                                                      void* __restrict__ out, DevStatus* st) {
    extern __shared__ __align__(16) int blk_smem[];
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    constexpr int nd = ND;   // 2 or 3 (template: no per-point dimension branches)
    const uint32_t bx = g.block[nd - 1], by = g.block[nd - 2], bz = nd == 3 ? g.block[0] : 1;
    const uint32_t per_warp = steps * (1 + (nd == 3 ? by : 0)) * 32;
    int* Gs = blk_smem + warp * per_warp + lane;   // [steps][32]: G of row y-1
    int* F0s = Gs + steps * 32;                    // [by][steps][32]: F of plane z-1 (3D)
    const uint64_t X = g.dims[nd - 1], Y = g.dims[nd - 2], Z = nd == 3 ? g.dims[0] : 1;
    const uint64_t sy = g.stride[nd - 2], sz = nd == 3 ? g.stride[0] : 0;
    const uint64_t nbx = g.nblk[nd - 1], nby = g.nblk[nd - 2], nbz = nd == 3 ? g.nblk[0] : 1;
    const uint64_t ntx = ceil_div(X, W), nyg = ceil_div(nby, nyb), ntask = ntx * nyg * nbz;
    const int r = (int)(cap >> 1);
    const bool seg0 = ONE ? lane % bx == 0 : lane == 0;   // block start (ONE) / first lane of a block row
    const unsigned upto = (2u << lane) - 1u;              // lanes 0..lane (lane 31: all)
    for (uint64_t t = blockIdx.x * (uint64_t)(blockDim.x >> 5) + warp; t < ntask;
         t += (uint64_t)gridDim.x * (blockDim.x >> 5)) {
        const uint64_t tx = t % ntx, t2 = t / ntx, cyg = t2 % nyg, cz = t2 / nyg;
        const uint64_t x0 = tx * W;
        const uint32_t lim = (uint32_t)umin(W, X - x0);   // valid columns of the strip
        const uint32_t nz = (uint32_t)umin(bz, Z - cz * bz);
        const uint64_t bcol = ONE ? (x0 + umin(lane, lim - 1)) / bx : x0 / bx;
        const uint64_t cy1 = umin(cyg * nyb + nyb, nby);
        for (uint64_t cy = cyg * nyb; cy < cy1; cy++) {
            const uint32_t ny = (uint32_t)umin(by, Y - cy * by);
            const uint64_t blk = (cz * nby + cy) * nbx + bcol;
            const bool skip = blockflag[blk] != 0;   // non-integer outlier: the fp64 replay owns it
            bool bad = false;
            // (z, y, s) iterations in groups of kRowPf: the group's codes are
            // loaded together (independent loads in flight) before the scans
            const uint32_t nit = nz * ny * steps;
            const uint64_t base = cz * bz * sz + cy * by * sy + x0;
            const uint64_t zjump = sz - (uint64_t)(ny - 1) * sy;   // row ny-1 of plane z -> row 0 of plane z+1
            uint64_t lrow = base, prow = base;
            uint32_t ls = 0, ly = 0, ps = 0, py = 0, pz = 0;
            int carry = 0;
            for (uint32_t it0 = 0; it0 < nit; it0 += kRowPf) {
                uint32_t cc[kRowPf];
#pragma unroll
                for (int k = 0; k < kRowPf; k++) {
                    const uint32_t c = ONE ? lane : ls * 32 + lane;
                    cc[k] = it0 + k < nit && c < lim ? (uint32_t)codes[lrow + c] : (uint32_t)r;
                    if (ONE || ++ls == steps) {
                        ls = 0;
                        if (++ly == ny) { ly = 0; lrow += zjump; } else lrow += sy;
                    }
                }
#pragma unroll
                for (int k = 0; k < kRowPf; k++) {
                    if (it0 + k >= nit) break;
                    const uint32_t s = ONE ? 0 : ps, y = py, z = pz;
                    const uint64_t rb = prow;
                    if (ONE || ++ps == steps) {
                        ps = 0;
                        if (++py == ny) { py = 0; pz++; prow += zjump; } else prow += sy;
                    }
                    const uint32_t c = s * 32 + lane;   // column within the strip
                    const bool valid = c < lim;
                    const uint32_t code = skip ? (uint32_t)r : cc[k];
                    const int Gp = y > 0 ? Gs[s * 32] : 0;
                    int* pf = F0s + (y * steps + s) * 32;
                    const int F0 = nd == 3 && z > 0 ? *pf : 0;
                    bool reset = ONE ? seg0 : (s == 0 && seg0);
                    int b = (int)code - r;
                    if (code == 0) {   // outlier: its final value is stored verbatim
                        const long long v = outlier_int(ol, rb + c);
                        const int Fv = (v < (1ll << 28) && v > -(1ll << 28)) ? (int)v : (1 << 29);
                        reset = true;
                        b = (int)((unsigned)Fv - (unsigned)F0 - (unsigned)Gp);
                    }
                    unsigned S = (unsigned)b;   // inclusive prefix sum of b
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const unsigned u = __shfl_up_sync(kFull, S, o);
                        if (lane >= (uint32_t)o) S += u;
                    }
                    const unsigned m = __ballot_sync(kFull, reset) & upto;
                    const int L = 31 - __clz((int)m);   // last reset lane at or left of this one
                    const unsigned Sx = __shfl_sync(kFull, S - (unsigned)b, L < 0 ? 0 : L);
                    const unsigned H = m ? S - Sx : (unsigned)carry + S;
                    if (!ONE) carry = (int)__shfl_sync(kFull, H, 31);
                    const int G = (int)(H + (unsigned)Gp);
                    const int F = (int)((unsigned)G + (unsigned)F0);
                    if (valid && !skip) {
                        bad |= !(F < (1 << 28) && F > -(1 << 28));
                        store_out<OUTK>(out, rb + c, F, two_eb);
                    }
                    Gs[s * 32] = G;
                    if (nd == 3) *pf = F;
                }
            }
            if (bad) {   // magnitude guard: the fp64 replay redoes the block
                blockflag[blk] = 1;
                atomicOr(&st->flags, (unsigned long long)F_OUT_SLOW);
            }
        }
    }
}

Geo make_geo(int ndims, const uint64_t dims[3], const uint32_t block[3]) {
    Geo g{};
    g.nd = ndims;
    for (int a = 0; a < 3; a++) {
        g.dims[a] = a < ndims ? dims[a] : 1;
        g.block[a] = a < ndims ? block[a] : 1;
        g.nblk[a] = a < ndims ? ceil_div(dims[a], block[a]) : 1;
    }
    g.stride[ndims - 1] = 1;
    for (int a = ndims - 2; a >= 0; a--) g.stride[a] = g.stride[a + 1] * g.dims[a + 1];
    for (int a = ndims; a < 3; a++) g.stride[a] = 1;
    return g;
}

}  // namespace

int launch_outlier_index(sdqz_ctx* ctx, const void* records, const uint64_t* idx, const double* val,
                         uint64_t k, uint64_t n, OutLookup* out) {
    int rc = SDQZ_OK;
    const uint64_t nb = ceil_div(n, 1024);
    unsigned long long* start = scratch_as<unsigned long long>(ctx, S_DENSE, nb + 2, &rc);
    if (!start) return rc;
    SDQZ_CUDA(ctx, cudaMemsetAsync(start + nb + 1, 0, 8, ctx->stream));
    const unsigned long long* rec = (const unsigned long long*)records;
    out->idx = rec ? rec : (const unsigned long long*)idx;
    out->val = rec ? rec + 1 : (const unsigned long long*)val;
    out->stride = rec ? 2 : 1;
    out->start = start;
    out->k = k;
    out->base = 0;
    out->big = start + nb + 1;
    uint64_t grid = ceil_div((nb + 1 > k ? nb + 1 : k), 256);
    if (grid > (uint64_t)ctx->num_sms * 8) grid = ctx->num_sms * 8;
    if (grid < 1) grid = 1;
    task_bounds_kernel<<<(unsigned)grid, 256, 0, ctx->stream>>>(out->idx, out->val, out->stride, k, nb, start);
    SDQZ_LAUNCHED_NAMED(ctx, "task_bounds_kernel");
    return SDQZ_OK;
}

int launch_outlier_scatter(sdqz_ctx* ctx, const void* records, const uint64_t* idx,
                           const double* val, uint64_t k, uint64_t n, const uint16_t* codes,
                           int ndims, const uint64_t dims[3], const uint32_t block[3],
                           uint8_t* blockflag, bool check_format) {
    (void)check_format;
    if (k == 0) return SDQZ_OK;
    Geo g = make_geo(ndims, dims, block);
    uint64_t grid = ceil_div(k, 256);
    if (grid > (uint64_t)ctx->num_sms * 8) grid = ctx->num_sms * 8;
    outlier_scatter_kernel<<<(unsigned)grid, 256, 0, ctx->stream>>>(
        (const unsigned long long*)records, idx, val, k, n, codes, g, blockflag, ctx->d_status, 0);
    SDQZ_LAUNCHED_NAMED(ctx, "outlier_scatter_kernel");
    return SDQZ_OK;
}

bool rq1d_records_ok(int ndims, const uint64_t dims[3], const uint32_t block[3], const void* codes,
                     const void* out, const void* records) {
    return records && ndims == 1 && block[0] == 32 && dims[0] >= 1 && ((uintptr_t)codes & 7) == 0 &&
           ((uintptr_t)out & 15) == 0 && !env_disabled("SDQZ_NO_VEC1D");
}

// 1D block-32 decompress tail: record checks (+ fp64-path blocks scattered),
// per-task record ranges, reconstruct from the records, fp64 replay of flagged blocks
int launch_reconstruct_1d_records(sdqz_ctx* ctx, const uint16_t* codes, const void* records, uint64_t k,
                                  uint64_t n, uint32_t cap, double two_eb, void* out, int out_kind,
                                  uint8_t* blockflag) {
    int rc = SDQZ_OK;
    const unsigned long long* rec = (const unsigned long long*)records;
    const uint64_t dims[3] = {n, 1, 1};
    const uint32_t block[3] = {32, 1, 1};
    Geo g = make_geo(1, dims, block);
    if (k) {
        uint64_t grid = ceil_div(k, 256);
        if (grid > (uint64_t)ctx->num_sms * 8) grid = ctx->num_sms * 8;
        outlier_scatter_kernel<<<(unsigned)grid, 256, 0, ctx->stream>>>(
            rec, nullptr, nullptr, k, n, codes, g, blockflag, ctx->d_status, 1);
        SDQZ_LAUNCHED_NAMED(ctx, "outlier_check_kernel");
    }
    // per-task record ranges = the lookup's 1024-point buckets (also serves the fp64 replay)
    const uint64_t ntask = ceil_div(n, 1024);
    OutLookup ol;
    if ((rc = launch_outlier_index(ctx, rec, nullptr, nullptr, k, n, &ol))) return rc;
    const unsigned long long* start = ol.start;
    uint64_t grid = ceil_div(ntask, kWarpsPerCta);
    if (grid > (uint64_t)ctx->num_sms * 8) grid = ctx->num_sms * 8;
    if (grid < 1) grid = 1;
    QualArgs qa;   // fused quality (sdqz_decompress_quality)
    if (ctx->qual.orig) {
        qa = ctx->qual;
        ctx->qual.nparts = grid;
    }
    if (out_kind == 0)
        rq1d_rec_kernel<0><<<(unsigned)grid, kThreads, 0, ctx->stream>>>(codes, rec, start, k, blockflag, n, cap,
                                                                       two_eb, out, ctx->d_status, qa);
    else
        rq1d_rec_kernel<1><<<(unsigned)grid, kThreads, 0, ctx->stream>>>(codes, rec, start, k, blockflag, n, cap,
                                                                       two_eb, out, ctx->d_status, qa);
    SDQZ_LAUNCHED_NAMED(ctx, "rq1d_rec_kernel");
    uint64_t gg = ceil_div(g.nblk[0], 128);
    if (gg > (uint64_t)ctx->num_sms) gg = ctx->num_sms;
    if (gg < 1) gg = 1;
    double* work = scratch_as<double>(ctx, S_WORK, gg * 128 * kSlotPts, &rc);
    if (!work) return rc;
    if (out_kind == 0)
        rq_generic_kernel<0><<<(unsigned)gg, 128, 0, ctx->stream>>>(codes, ol, blockflag, 1,
                                                                  g, cap, two_eb, work, out, ctx->d_status, kSlotPts);
    else
        rq_generic_kernel<1><<<(unsigned)gg, 128, 0, ctx->stream>>>(codes, ol, blockflag, 1,
                                                                  g, cap, two_eb, work, out, ctx->d_status, kSlotPts);
    SDQZ_LAUNCHED_NAMED(ctx, "rq_generic_kernel");
    return SDQZ_OK;
}

int launch_count_zero(sdqz_ctx* ctx, const uint16_t* codes, uint64_t n) {
    uint64_t grid = ceil_div(n, 256);
    if (grid > (uint64_t)ctx->num_sms * 8) grid = ctx->num_sms * 8;
    if (grid < 1) grid = 1;
    count_zero_kernel<<<(unsigned)grid, 256, 0, ctx->stream>>>(codes, n, ctx->d_status);
    SDQZ_LAUNCHED_NAMED(ctx, "count_zero_kernel");
    return SDQZ_OK;
}

int launch_narrow_codes(sdqz_ctx* ctx, const uint32_t* in, uint64_t n, uint32_t cap, uint16_t* out) {
    uint64_t grid = ceil_div(n, 256);
    if (grid > (uint64_t)ctx->num_sms * 8) grid = ctx->num_sms * 8;
    if (grid < 1) grid = 1;
    narrow_codes_kernel<<<(unsigned)grid, 256, 0, ctx->stream>>>(in, n, cap, out, ctx->d_status);
    SDQZ_LAUNCHED_NAMED(ctx, "narrow_codes_kernel");
    return SDQZ_OK;
}

int launch_reconstruct(sdqz_ctx* ctx, const uint16_t* codes, const OutLookup& ol,
                       const uint8_t* blockflag, bool any_slow, int ndims, const uint64_t dims[3],
                       const uint32_t block[3], uint32_t cap, double two_eb, void* out,
                       int out_kind) {
    int rc = SDQZ_OK;
    Geo g = make_geo(ndims, dims, block);
    const OutLookup dn = ol;
    uint64_t n = g.dims[0] * g.dims[1] * g.dims[2];
    int max_grid = ctx->num_sms * 8;
    bool fast = is_fast_shape(ndims, block);
    if (fast) {
        uint64_t ntask;
        if (ndims == 3) ntask = ceil_div(ceil_div(dims[2], 8), 4) * ceil_div(dims[1], 8) * ceil_div(dims[0], 8);
        else if (ndims == 2) ntask = ceil_div(ceil_div(dims[1], 16), 2) * ceil_div(dims[0], 16);
        else ntask = ceil_div(dims[0], 32);
        uint64_t grid = ceil_div(ntask, kWarpsPerCta);
        if (grid > (uint64_t)max_grid) grid = max_grid;
        if (grid < 1) grid = 1;
        int slow = any_slow ? 1 : 0;
        // cp.async staging needs 4-byte aligned code rows
        const uint64_t nblk3 = ndims == 3 ? ceil_div(dims[0], 8) * ceil_div(dims[1], 8) * ceil_div(dims[2], 8) : 1;
        uint64_t bgrid = ceil_div(nblk3, 64);
        if (bgrid > (uint64_t)ctx->num_sms * 16) bgrid = (uint64_t)ctx->num_sms * 16;
        // vectorised 2D: 16 x 128 tasks (8-byte code rows, 16-byte output rows)
        const bool vec2d = ndims == 2 && dims[1] % 4 == 0 && ((uintptr_t)codes & 7) == 0 &&
                           ((uintptr_t)out & 15) == 0 && !env_disabled("SDQZ_NO_VEC2D");
        uint64_t grid2 = ndims == 2 ? ceil_div(ceil_div(dims[1], 128) * ceil_div(dims[0], 16), kWarpsPerCta) : 1;
        if (grid2 > (uint64_t)ctx->num_sms * 8) grid2 = (uint64_t)ctx->num_sms * 8;
        if (grid2 < 1) grid2 = 1;
        // vectorised 1D: whole 1024-point tasks (8-byte code rows, 16-byte output rows)
        const bool vec1d = ndims == 1 && dims[0] >= 1024 && ((uintptr_t)codes & 7) == 0 &&
                           ((uintptr_t)out & 15) == 0 && !env_disabled("SDQZ_NO_VEC1D");
        const uint64_t nt1 = ndims == 1 ? dims[0] / 1024 : 0, off1 = nt1 * 1024;
        uint64_t vgrid = ceil_div(nt1, kWarpsPerCta);
        if (vgrid > (uint64_t)ctx->num_sms * 8) vgrid = (uint64_t)ctx->num_sms * 8;
        if (vgrid < 1) vgrid = 1;
        // fused quality: the 3D block and vectorised 2D kernels (any other path
        // leaves nparts = 0 and the caller scores in a separate pass)
        QualArgs qa;
        if (ctx->qual.orig && (ndims == 3 || vec2d)) {
            qa = ctx->qual;
            ctx->qual.nparts = ndims == 3 ? bgrid : grid2;
        }
        OutLookup dn_tail = ol;   // the 1D tail kernel indexes from off1
        dn_tail.base += off1;
#define RQ_LAUNCH(K)                                                                                 \
        if (ndims == 3)                                                                              \
            rq3d_block_kernel<K><<<(unsigned)bgrid, 64, 0, ctx->stream>>>(codes, dn, const_cast<uint8_t*>(blockflag), slow, \
                                                                        dims[0], dims[1], dims[2], cap, two_eb, out, ctx->d_status, qa); \
        else if (vec2d)                                                                              \
            rq2d_vec_kernel<K><<<(unsigned)grid2, kThreads, 0, ctx->stream>>>(codes, dn, blockflag, slow, \
                                                                             dims[0], dims[1], cap, two_eb, out, qa); \
        else if (ndims == 2)                                                                         \
            rq2d_kernel<K><<<(unsigned)grid, kThreads, 0, ctx->stream>>>(codes, dn, blockflag, slow,   \
                                                                        dims[0], dims[1], cap, two_eb, out); \
        else if (vec1d) {                                                                            \
            rq1d_vec_kernel<K><<<(unsigned)vgrid, kThreads, 0, ctx->stream>>>(codes, dn, blockflag, slow, \
                                                                             nt1, cap, two_eb, out); \
            if (off1 < dims[0])                                                                      \
                rq1d_kernel<K><<<1, kThreads, 0, ctx->stream>>>(codes + off1, dn_tail,              \
                    blockflag + off1 / 32, slow, dims[0] - off1, cap, two_eb,                        \
                    (char*)out + off1 * (K == 0 ? 4 : 8));                                           \
        } else                                                                                       \
            rq1d_kernel<K><<<(unsigned)grid, kThreads, 0, ctx->stream>>>(codes, dn, blockflag, slow,   \
                                                                        dims[0], cap, two_eb, out);
        if (out_kind == 0) { RQ_LAUNCH(0) } else { RQ_LAUNCH(1) }
#undef RQ_LAUNCH
        if (ndims == 3) SDQZ_LAUNCHED_NAMED(ctx, "rq3d_block_kernel");
        else if (ndims == 2) SDQZ_LAUNCHED_NAMED(ctx, vec2d ? "rq2d_vec_kernel" : "rq2d_kernel");
        else SDQZ_LAUNCHED_NAMED(ctx, vec1d ? "rq1d_vec_kernel" : "rq1d_kernel");
        if (!any_slow) return SDQZ_OK;
    }
    // generic shapes: thread per block (int32 recurrence) unless the per-thread
    // slots or the replay slots get too large
    uint64_t bpts = 1;
    for (int a = 0; a < ndims; a++) bpts *= block[a];
    const uint32_t slots = blk_slots(ndims, g.block);
    const bool blk = !fast && slots <= kBlkMaxSlots && bpts <= 65536 && !env_disabled("SDQZ_NO_BLK");
    uint64_t nblocks = g.nblk[0] * g.nblk[1] * g.nblk[2];
    // 2D / 3D row kernel: strips of 32 / bx whole blocks (bx <= 32) or one
    // block in ceil(bx / 32) lane segments; lane-private slots <= 12 KB a warp
    const uint32_t bxx = block[ndims - 1];
    const uint32_t rw = bxx <= 32 ? (32 / bxx) * bxx : bxx, rsteps = (rw + 31) / 32;
    const char* rows_env = getenv("SDQZ_RQ_ROWS");   // 0 | 1: force off / on (tests)
    const bool rows_ok = ndims >= 2 && (uint64_t)rsteps * (1 + (ndims == 3 ? block[ndims - 2] : 0)) <= 96 &&
                         (rows_env ? rows_env[0] == '1' : bpts >= 128);
    if (blk && ndims == 1 && block[0] >= 32) {   // long 1D blocks: warp-wide scans over tasks of whole blocks
        const uint64_t task = (uint64_t)block[0] * ceil_div(1024, block[0]);
        const int narrow_ok = (uint64_t)block[0] * (cap >> 1) < (1ull << 29) ? 1 : 0;   // int32 F bound
        uint64_t bg = ceil_div(ceil_div(n, task), 8);
        if (bg > (uint64_t)ctx->num_sms * 16) bg = (uint64_t)ctx->num_sms * 16;
        if (bg < 1) bg = 1;
        if (out_kind == 0)
            rq1d_seg_kernel<0><<<(unsigned)bg, 256, 0, ctx->stream>>>(codes, dn, n, block[0], task, cap, two_eb, out,
                                                                     narrow_ok);
        else
            rq1d_seg_kernel<1><<<(unsigned)bg, 256, 0, ctx->stream>>>(codes, dn, n, block[0], task, cap, two_eb, out,
                                                                     narrow_ok);
        SDQZ_LAUNCHED_NAMED(ctx, "rq1d_seg_kernel");
    } else if (blk && ndims >= 2 && rows_ok) {   // warp per strip of block columns, lane = column
        // block rows per task: >= 32 row iterations a warp task
        const uint64_t iters = (uint64_t)rsteps * block[ndims - 2] * (ndims == 3 ? block[0] : 1);
        const uint32_t nyb = iters >= 32 ? 1 : (uint32_t)ceil_div(32, iters);
        const uint64_t ntask = ceil_div(g.dims[ndims - 1], rw) * ceil_div(g.nblk[ndims - 2], nyb) *
                               (ndims == 3 ? g.nblk[0] : 1);
        uint64_t bg = ceil_div(ntask, 8);
        if (bg > (uint64_t)ctx->num_sms * 16) bg = (uint64_t)ctx->num_sms * 16;
        if (bg < 1) bg = 1;
        const size_t dsm = (size_t)8 * rsteps * (1 + (ndims == 3 ? block[ndims - 2] : 0)) * 32 * 4;
#define RQ_ROWS(K, ONE, ND)                                                                                   \
        ensure_smem(ctx, (const void*)rq_rows_kernel<K, ONE, ND>, dsm);                                       \
        rq_rows_kernel<K, ONE, ND><<<(unsigned)bg, 256, dsm, ctx->stream>>>(codes, dn, const_cast<uint8_t*>(blockflag), \
                                                                          g, rw, rsteps, nyb, cap, two_eb, out, ctx->d_status);
#define RQ_ROWS_ND(K, ONE) if (ndims == 3) { RQ_ROWS(K, ONE, 3) } else { RQ_ROWS(K, ONE, 2) }
        if (out_kind == 0) {
            if (rsteps == 1) { RQ_ROWS_ND(0, true) } else { RQ_ROWS_ND(0, false) }
        } else {
            if (rsteps == 1) { RQ_ROWS_ND(1, true) } else { RQ_ROWS_ND(1, false) }
        }
#undef RQ_ROWS_ND
#undef RQ_ROWS
        SDQZ_LAUNCHED_NAMED(ctx, "rq_rows_kernel");
    } else if (blk) {
        const uint32_t T = slots * 4 <= 1024 ? 64 : 32;
        const size_t dsm = (size_t)T * slots * 4;
        uint64_t bg = ceil_div(nblocks, T);
        if (bg > (uint64_t)ctx->num_sms * 64) bg = (uint64_t)ctx->num_sms * 64;
        if (bg < 1) bg = 1;
#define RQ_BLOCKS(K, ND)                                                                                  \
        ensure_smem(ctx, (const void*)rq_blocks_kernel<K, ND>, dsm);                                      \
        rq_blocks_kernel<K, ND><<<(unsigned)bg, T, dsm, ctx->stream>>>(codes, dn, const_cast<uint8_t*>(blockflag), g, \
                                                                     cap, two_eb, out, ctx->d_status);
#define RQ_BLOCKS_ND(K) if (ndims == 3) { RQ_BLOCKS(K, 3) } else if (ndims == 2) { RQ_BLOCKS(K, 2) } else { RQ_BLOCKS(K, 0) }
        if (out_kind == 0) { RQ_BLOCKS_ND(0) } else { RQ_BLOCKS_ND(1) }
#undef RQ_BLOCKS_ND
#undef RQ_BLOCKS
        SDQZ_LAUNCHED_NAMED(ctx, "rq_blocks_kernel");
    }
    const bool only_flagged = fast || blk;
    uint64_t grid = ceil_div(nblocks, 128);
    // flagged-blocks-only replay: usually nothing to do (the kernel exits on
    // the status word), so one CTA per SM bounds the idle launch cost
    if (only_flagged && grid > (uint64_t)ctx->num_sms) grid = ctx->num_sms;
    if (grid > (uint64_t)max_grid) grid = max_grid;
    if (grid < 1) grid = 1;
    // whole-field fp64 scratch for the all-blocks replay; per-thread block slots otherwise
    // (at most ~512 MB of slots: fewer replay threads for big blocks)
    const uint64_t slot_pts = bpts > kSlotPts ? bpts : kSlotPts;
    if (only_flagged) {
        const uint64_t max_threads = std::max<uint64_t>(128, (512ull << 20) / 8 / slot_pts);
        if (grid * 128 > max_threads) grid = std::max<uint64_t>(1, max_threads / 128);
    }
    double* work = scratch_as<double>(ctx, S_WORK, only_flagged ? grid * 128 * slot_pts : n, &rc);
    if (!work) return rc;
    int only = only_flagged ? 1 : 0;
    if (out_kind == 0)
        rq_generic_kernel<0><<<(unsigned)grid, 128, 0, ctx->stream>>>(codes, dn, blockflag, only, g, cap,
                                                                    two_eb, work, out, ctx->d_status, slot_pts);
    else
        rq_generic_kernel<1><<<(unsigned)grid, 128, 0, ctx->stream>>>(codes, dn, blockflag, only, g, cap,
                                                                    two_eb, work, out, ctx->d_status, slot_pts);
    SDQZ_LAUNCHED_NAMED(ctx, "rq_generic_kernel");
    return SDQZ_OK;
}

}  // namespace sdqz
