// dualquant.cu -- K2: fused prequantization + blockwise Lorenzo postquantization
// + quant-code histogram (dualquant.py:62-194, huffman.py:77-95).
//
// Layout: the field is row-major (axis 0 slowest).  A warp owns a "task" of
// 512 points -- 3D: 4 blocks of 8x8x8 side by side along x (lane = x), the
// warp walks the 8 planes x 8 rows; 2D: 2 blocks of 16x16 (lane = x, walks 16
// rows); 1D: 16 consecutive blocks of 32 (lane = position in block).  Every
// warp load/store is one contiguous 128 B (fp32 in) / 64 B (u16 codes) row
// segment, so the kernel streams 4N + 2N bytes at HBM rate.
//
// Arithmetic.  Prequantization is IEEE fp64 division + floor(|x|+.5) +
// copysign exactly as dualquant.py:76-77.  The Lorenzo residual is computed
// in int32 as D_z D_y D_x d (finite differences, one shuffle per point) when
// every prequantized value of the warp's task is below 2^27 in magnitude
// (then all partial sums are exact integers and equal the reference's fp64
// result); otherwise the warp recomputes its task in fp64 with the reference's
// 7-term order (dualquant.py:125-129), which is bit-exact for any magnitude.
// Non-default block shapes take a generic one-thread-per-point fp64 kernel.
//
// Histogram: 16 bins around the radius are counted in packed 8-bit register
// counters (two u64 per thread, flushed per task with __reduce_add_sync);
// codes outside that window use shared-memory atomics; each CTA merges its
// shared histogram into the global uint64 histogram once.
#include <type_traits>
#include "kernels.cuh"
#include "tma.cuh"

namespace sdqz {

namespace {

constexpr int kThreads = 256;
constexpr int kWarpsPerCta = kThreads / 32;
constexpr uint32_t kSmemHistMax = 16384;   // caps above this count in global memory

struct HistCtx {
    uint32_t* shist;                 // shared (or null => global)
    unsigned long long* ghist;       // global uint64[cap] (may be null: no histogram)
    uint32_t cap, wbase;             // window = [wbase, wbase + 16)
    unsigned long long lo, hi;       // packed 8-bit counters
};

__device__ __forceinline__ void hist_add(HistCtx& h, uint32_t code) {
    uint32_t dw = code - h.wbase;
    if (dw < 16u) {
        unsigned long long inc = 1ull << (8 * (dw & 7));
        if (dw < 8) h.lo += inc; else h.hi += inc;
    } else if (h.shist) {
        atomicAdd(&h.shist[code], 1u);
    } else if (h.ghist) {
        atomicAdd(&h.ghist[code], 1ull);
    }
}

__device__ __forceinline__ void hist_flush(HistCtx& h) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
        uint32_t c = (uint32_t)(((k < 8) ? (h.lo >> (8 * k)) : (h.hi >> (8 * (k - 8)))) & 0xFF);
        uint32_t s = __reduce_add_sync(kFull, c);
        if (s && lane_id() == 0) {
            uint32_t bin = h.wbase + k;
            if (h.shist) atomicAdd(&h.shist[bin], s);
            else if (h.ghist) atomicAdd(&h.ghist[bin], (unsigned long long)s);
        }
    }
    h.lo = h.hi = 0;
}

template <int KIND>
__device__ __forceinline__ double load_q(const void* in, uint64_t i, double two_eb, bool& bad) {
    double v;
    if (KIND == 0) v = (double)__ldg((const float*)in + i);
    else v = __ldg((const double*)in + i);
    bad |= !isfinite(v);
    return KIND == 2 ? v : prequant(v, two_eb);
}

// load_q for one thread (no warp vote): fp32 input by the reciprocal multiply
// of prequant_int_fast with the same tie window; a value inside it, at or
// above 2^27 units, or non-finite takes the exact division
template <int KIND>
__device__ __forceinline__ double load_q_fast(const void* in, uint64_t i, double two_eb, double rcp, bool& bad) {
    if (KIND != 0) return load_q<KIND>(in, i, two_eb, bad);
    const float v = __ldg((const float*)in + i);
    bad |= !isfinite(v);
    const double y = __dmul_rn((double)v, rcp);
    const double ay = fabs(y);
    if (ay < 134217728.0) {
        const double t = __dadd_rn(ay, 0.5);
        const double fl = floor(t);
        const double fr = __dsub_rn(t, fl);
        if (fr >= 2.384185791015625e-07 && fr <= 1.0 - 2.384185791015625e-07) return copysign(fl, y);
    }
    return prequant((double)v, two_eb);
}

__device__ __forceinline__ uint32_t code_of_int(int delta, int r) {
    return (delta > -r && delta < r) ? (uint32_t)(delta + r) : 0u;
}
__device__ __forceinline__ uint32_t code_of_f64(double delta, int r) {
    return (delta > (double)-r && delta < (double)r) ? (uint32_t)__dadd_rn(delta, (double)r) : 0u;
}

__device__ __forceinline__ void hist_init(HistCtx& h, uint32_t* smem, unsigned long long* ghist,
                                          uint32_t cap) {
    h.ghist = ghist;
    h.cap = cap;
    h.shist = (ghist && cap <= kSmemHistMax) ? smem : nullptr;
    h.wbase = cap >= 16 ? cap / 2 - 8 : 0;
    h.lo = h.hi = 0;
    if (h.shist) {
        for (uint32_t i = threadIdx.x; i < cap; i += blockDim.x) h.shist[i] = 0;
    }
    __syncthreads();
}

__device__ __forceinline__ void hist_finish(HistCtx& h) {
    __syncthreads();
    if (h.shist) {
        for (uint32_t i = threadIdx.x; i < h.cap; i += blockDim.x) {
            uint32_t c = h.shist[i];
            if (c) atomicAdd(&h.ghist[i], (unsigned long long)c);
        }
    }
}

// ----------------------------------------------------------------------------
// Task loading.  fp32 input: all of a task's values are loaded up front (one
// coalesced 128 B row per load, 16-64 loads in flight per warp) and kept as
// floats; a conservative bound max|x| / 2eb < 2^27 - 4 decides, per warp,
// whether the exact int32 path applies (then every |d| < 2^27).  fp64 input
// is loaded row by row (register budget) and always takes the fp64 path
// check per value.
// ----------------------------------------------------------------------------
template <int KIND>
struct Raw { using T = double; };
template <>
struct Raw<0> { using T = float; };

template <int KIND>
__device__ __forceinline__ typename Raw<KIND>::T load_raw(const void* in, uint64_t i) {
    if (KIND == 0) return __ldg((const float*)in + i);
    return __ldg((const double*)in + i);
}

template <int KIND>
__device__ __forceinline__ double to_q(typename Raw<KIND>::T v, double two_eb) {
    return KIND == 2 ? (double)v : prequant((double)v, two_eb);
}

constexpr double kIntBound = 134217724.0;   // 2^27 - 4

// fp64 task in the reference's term order (dualquant.py:125-129):
// +(z-1,y,x) +(z,y-1,x) +(z,y,x-1) -(z-1,y-1,x) -(z-1,y,x-1) -(z,y-1,x-1) +(z-1,y-1,x-1).
// Out of line so its registers do not inflate the int32 fast path; called
// warp-uniformly, it counts into its own window and flushes before returning.
template <int KIND>
__device__ __noinline__ void dq3d_task_f64(const void* __restrict__ in, uint64_t base, uint64_t YX,
                                           uint64_t X, bool xin, int nz, int ny, uint32_t xl,
                                           double two_eb, int r, uint16_t* __restrict__ codes,
                                           HistCtx hc, bool& bad) {
    using T = typename Raw<KIND>::T;
    HistCtx h = hc;
    h.lo = h.hi = 0;
    double P[8];
#pragma unroll
    for (int y = 0; y < 8; y++) P[y] = 0.0;
    for (int z = 0; z < 8; z++) {
        double cprev = 0.0, pold = 0.0;
#pragma unroll
        for (int y = 0; y < 8; y++) {
            double q = 0.0;
            if (xin && z < nz && y < ny) {
                T v = load_raw<KIND>(in, base + z * YX + y * X);
                bad |= !isfinite((double)v);
                q = to_q<KIND>(v, two_eb);
            }
            const double pz = P[y];
            const double pzm = pold;           // P_old[y-1] (0 for y == 0)
            const double cm = cprev;           // (z, y-1, x)  (0 for y == 0)
            double n_c = __shfl_up_sync(kFull, q, 1);
            double n_pz = __shfl_up_sync(kFull, pz, 1);
            double n_cm = __shfl_up_sync(kFull, cm, 1);
            double n_pzm = __shfl_up_sync(kFull, pzm, 1);
            if (!xl) n_c = n_pz = n_cm = n_pzm = 0.0;
            double pred = __dadd_rn(pz, cm);
            pred = __dadd_rn(pred, n_c);
            pred = __dsub_rn(pred, pzm);
            pred = __dsub_rn(pred, n_pz);
            pred = __dsub_rn(pred, n_cm);
            pred = __dadd_rn(pred, n_pzm);
            const double delta = __dsub_rn(q, pred);
            pold = pz;
            P[y] = q;
            cprev = q;
            if (xin && z < nz && y < ny) {
                uint32_t c = code_of_f64(delta, r);
                codes[base + z * YX + y * X] = (uint16_t)c;
                hist_add(h, c);
            }
        }
    }
    hist_flush(h);
}

// ----------------------------------------------------------------------------
// 3D, block 8x8x8
// ----------------------------------------------------------------------------
template <int KIND>
__global__ void __launch_bounds__(kThreads, 2) dq3d_kernel(const void* __restrict__ in, uint64_t Z,
                                                           uint64_t Y, uint64_t X, uint32_t cap,
                                                           DevStatus* st, uint16_t* __restrict__ codes,
                                                           unsigned long long* ghist) {
    using T = typename Raw<KIND>::T;
    extern __shared__ uint32_t smem_hist[];
    HistCtx h;
    hist_init(h, smem_hist, ghist, cap);
    const double two_eb = st->two_eb;
    const double rcp = __drcp_rn(two_eb);
    const int r = (int)(cap >> 1);
    const uint32_t lane = lane_id(), xl = lane & 7;
    const uint64_t nbx4 = ceil_div(ceil_div(X, 8), 4), nby = ceil_div(Y, 8), nbz = ceil_div(Z, 8);
    const uint64_t ntask = nbx4 * nby * nbz;
    const uint64_t YX = Y * X;
    bool bad = false;
    for (uint64_t task = blockIdx.x * (uint64_t)kWarpsPerCta + (threadIdx.x >> 5); task < ntask;
         task += (uint64_t)gridDim.x * kWarpsPerCta) {
        const uint64_t bx4 = task % nbx4, t2 = task / nbx4;
        const uint64_t by = t2 % nby, bz = t2 / nby;
        const uint64_t x = bx4 * 32 + lane, y0 = by * 8, z0 = bz * 8;
        const bool xin = x < X;
        const int ny = (int)umin(8, Y - y0), nz = (int)umin(8, Z - z0);
        const uint64_t base = z0 * YX + y0 * X + x;
        bool use_int = false;
        if (KIND == 0) {
            float raw[8][8];
            float mx = 0.f;
#pragma unroll
            for (int z = 0; z < 8; z++)
#pragma unroll
                for (int y = 0; y < 8; y++) {
                    float v = 0.f;
                    if (xin && z < nz && y < ny) v = load_raw<0>(in, base + z * YX + y * X);
                    raw[z][y] = v;
                    mx = fmaxf(mx, fabsf(v));   // NaN -> ignored by fmaxf; flagged below
                    bad |= !isfinite(v);
                }
            use_int = __all_sync(kFull, !bad && (double)mx / two_eb < kIntBound);
            if (use_int) {
#pragma unroll
                for (int z = 0; z < 8; z++)
#pragma unroll
                    for (int y = 0; y < 8; y++)
                        raw[z][y] = __int_as_float(prequant_int(raw[z][y], rcp, two_eb));
                int hprev[8];
#pragma unroll
                for (int z = 0; z < 8; z++) {
                    int gprev = 0;
#pragma unroll
                    for (int y = 0; y < 8; y++) {
                        int v = __float_as_int(raw[z][y]);
                        int left = __shfl_up_sync(kFull, v, 1);
                        int g = v - (xl ? left : 0);
                        int hh = g - gprev;
                        gprev = g;
                        int delta = hh - (z ? hprev[y] : 0);
                        hprev[y] = hh;
                        if (xin && z < nz && y < ny) {
                            uint32_t c = code_of_int(delta, r);
                            codes[base + z * YX + y * X] = (uint16_t)c;
                            hist_add(h, c);
                        }
                    }
                }
            }
        }
        if (!use_int) dq3d_task_f64<KIND>(in, base, YX, X, xin, nz, ny, xl, two_eb, r, codes, h, bad);
        hist_flush(h);
    }
    if (__any_sync(kFull, bad) && lane == 0) atomicOr(&st->flags, (unsigned long long)F_NONFINITE);
    hist_finish(h);
}

// ----------------------------------------------------------------------------
// 3D, block 8x8x8, fp32 input staged by TMA.  Each warp streams its own tasks
// (4 blocks side by side along x, lane = x) through a 3-stage ring of
// 32 x 8 x 2 tiles (OOB zero-filled by the TMA unit): the next two plane
// pairs are in flight while one is computed from shared memory.
//
// Prequantization in fixed point.  One fp64 FMA  R = v * RN(1/2eb) + C  with
// C = 1.5 * 2^30 + 0.5 + 2^-21 stays in the binade [2^30, 2^31) whenever
// |v / 2eb| < 2^29, where the ulp is 2^-22: the mantissa holds
// x = round((v/2eb + 0.5) * 2^22) + 2^51 + 2 as an integer, so the rounded
// quotient is bits [22, 51) of R plus a constant bias K (one funnel shift, no
// float->int conversion, no sign handling: the bias cancels in the Lorenzo
// differences and is subtracted only at the x edge of a block).  The FMA is
// within 0.57 units of 2^-22 of the exact value, so the result can differ
// from the reference's copysign(floor(RN(RN(|v| / 2eb) + 0.5)), v) only when
// x mod 2^22 < 4 (a value within a few 2^-22 of a rounding tie, probability
// ~1e-6).  Such values are redone in place with exact division (one warp vote
// per plane).  Any |v / 2eb| >= 2^27 - 2048 (high word of R outside the
// bound; includes NaN/Inf) marks the task; a marked task's counts are taken
// back and it is redone in fp64 with exact division in the reference's term
// order.
//
// D_x D_y D_z are int32 differences (exact below 2^27); the code and its
// histogram bin follow.  The 16 bins around the radius are lane-private
// shared counters ([warp][bin][lane]: bank = lane, conflict-free), other
// codes go to the CTA histogram: one red.shared per point either way.
// ----------------------------------------------------------------------------
constexpr int kTmaWarps = 8;
constexpr int kStages = 3;                       // ring of plane-pair tiles per warp
constexpr uint32_t kPair = 32 * 8 * 2;           // floats per stage: 32 x, 8 y, 2 z
constexpr uint32_t kHot = 16;                    // lane-private bins per warp
constexpr double kFixC = 1610612736.0 + 0.5 + 4.76837158203125e-07;   // 1.5*2^30 + 0.5 + 2^-21
constexpr double kFixBound = 134215680.0;                             // 2^27 - 2048
constexpr int kFixK = 0x60000000;   // bits [22, 53) of C - 0.5 - 2^-21 (exponent bit 52 + 2^51)

// hot bin of code c for this lane: hb + 128c (hb = lane base - 128 wbase)
__device__ __forceinline__ void hot_add(uint32_t hb, uint32_t c, uint32_t wbase, HistCtx& h, int by) {
    if (c - wbase < kHot) {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(hb + c * 128u), "r"(by) : "memory");
    } else if (h.shist) {
        atomicAdd(&h.shist[c], (uint32_t)by);
    } else if (h.ghist) {
        atomicAdd(&h.ghist[c], (unsigned long long)(long long)by);
    }
}

// take back the counts of a task's fast-path codes (read back from global
// memory: each lane reads the column it wrote)
__device__ __noinline__ void dq3d_uncount(const uint16_t* __restrict__ codes, uint64_t base, uint64_t YX,
                                          uint64_t X, bool xin, int nz, int ny, uint32_t hb,
                                          uint32_t wbase, HistCtx h) {
    if (!xin) return;
    for (int z = 0; z < nz; z++)
        for (int y = 0; y < ny; y++) hot_add(hb, codes[base + z * YX + y * X], wbase, h, -1);
}

__device__ __forceinline__ uint16_t* row_ptr(uint16_t* p, uint32_t rowbytes, uint32_t y) {
    return (uint16_t*)((char*)p + (y * rowbytes));
}

// one plane pair (2 z x 8 y) of a task.  FULL: every point is inside the
// field (no predicates); SH: the CTA histogram is in shared memory.
template <bool FULL, bool SH>
__device__ __forceinline__ void dq3d_pair(const float* __restrict__ tile, uint32_t lane, uint32_t xl,
                                          double rcp, double two_eb, uint32_t hi_lo, uint32_t hi_span, int r, uint32_t wbase,
                                          uint32_t hb, uint32_t shist_s, HistCtx& h, int (&hprev)[8],
                                          bool& mark, uint16_t* tbz0, uint16_t* tbz1, uint32_t rowbytes,
                                          bool zin0, bool zin1, int ny) {
    // phases keep the 8 rows of a plane independent until the y recurrence:
    // loads / prequantization / shuffles of all rows are in flight together
#pragma unroll
    for (int zz = 0; zz < 2; zz++) {
        uint16_t* const tbz = zz ? tbz1 : tbz0;
        const bool zin = zz ? zin1 : zin0;
        int qv[8], left[8];   // rounded quotients + kFixK
        bool amb = false;
#pragma unroll
        for (int y = 0; y < 8; y++) {
            const float v = tile[(zz * 8 + y) * 32 + lane];
            const double R = __fma_rn((double)v, rcp, kFixC);
            const uint32_t lo = (uint32_t)__double2loint(R), hi = (uint32_t)__double2hiint(R);
            amb |= (lo & 0x3FFFFCu) == 0u;
            mark |= (hi - hi_lo) >= hi_span;
            qv[y] = (int)__funnelshift_r(lo, hi, 22);
        }
        if (__any_sync(kFull, amb)) {   // rare: exact division near a rounding tie
#pragma unroll
            for (int y = 0; y < 8; y++) {
                const float v = tile[(zz * 8 + y) * 32 + lane];
                const double R = __fma_rn((double)v, rcp, kFixC);
                if (((uint32_t)__double2loint(R) & 0x3FFFFCu) == 0u) {
                    const int m = (int)floor(__dadd_rn(fabs(__ddiv_rn((double)v, two_eb)), 0.5));
                    qv[y] = (v < 0.f ? -m : m) + kFixK;
                }
            }
        }
#pragma unroll
        for (int y = 0; y < 8; y++) left[y] = __shfl_up_sync(kFull, qv[y], 1);
        int gprev = 0;
        uint32_t cc[8];
#pragma unroll
        for (int y = 0; y < 8; y++) {
            const int g = qv[y] - (xl ? left[y] : kFixK);
            const int hh = g - gprev;
            gprev = g;
            const uint32_t uu = (uint32_t)(hh - hprev[y] + r);
            hprev[y] = hh;
            cc[y] = (uu - 1u) < (uint32_t)(2 * r - 1) ? uu : 0u;   // -r < delta < r
        }
#pragma unroll
        for (int y = 0; y < 8; y++) {
            const uint32_t c = cc[y];
            if (FULL || (zin && y < ny)) {
                *row_ptr(tbz, rowbytes, (uint32_t)y) = (uint16_t)c;
                if (SH) {   // one shared reduction: lane-private hot bin or CTA bin
                    const bool hot = c - wbase < kHot;
                    const uint32_t addr = c * (hot ? 128u : 4u) + (hot ? hb : shist_s);
                    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
                } else {
                    hot_add(hb, c, wbase, h, 1);
                }
            }
        }
    }
}

__global__ void __launch_bounds__(kTmaWarps * 32, 2) dq3d_tma_kernel(
    const __grid_constant__ CUtensorMap tmap, const float* __restrict__ in, uint64_t Z, uint64_t Y,
    uint64_t X, uint32_t cap, DevStatus* st, uint16_t* __restrict__ codes,
    unsigned long long* ghist) {
    extern __shared__ __align__(128) unsigned char dsm[];
    float* tiles = reinterpret_cast<float*>(dsm);                              // [warp][stage][kPair]
    uint64_t* bars = reinterpret_cast<uint64_t*>(dsm + kTmaWarps * kStages * kPair * 4);
    uint32_t* hot = reinterpret_cast<uint32_t*>(bars + kTmaWarps * kStages);   // [warp][kHot][32]
    uint32_t* shist_base = hot + kTmaWarps * kHot * 32;
    for (uint32_t i = threadIdx.x; i < kTmaWarps * kHot * 32; i += blockDim.x) hot[i] = 0;
    HistCtx h;
    hist_init(h, shist_base, ghist, cap);   // (syncs)
    const double two_eb = st->two_eb;
    const double rcp = __drcp_rn(two_eb);
    // in bounds: hi(C - B) < hi(R) < hi(C + B), one unsigned compare
    const uint32_t hi_lo = (uint32_t)__double2hiint(kFixC - kFixBound) + 1u;
    const uint32_t hi_span = (uint32_t)__double2hiint(kFixC + kFixBound) - hi_lo;
    const int r = (int)(cap >> 1);
    const uint32_t wbase = cap >= 2 * kHot ? (uint32_t)r - kHot / 2 : 0u;
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5, xl = lane & 7;
    const uint32_t hb = smem_u32(hot + wid * kHot * 32 + lane) - wbase * 128u;
    // task indices and in-task offsets fit 32 bits (TMA extents < 2^31, a task
    // spans < 8 planes): 32-bit index math
    const uint32_t nbx4 = (uint32_t)ceil_div(ceil_div(X, 8), 4), nby = (uint32_t)ceil_div(Y, 8),
                   nbz = (uint32_t)ceil_div(Z, 8);
    const uint32_t ntask = nbx4 * nby * nbz;
    const uint64_t YX = Y * X;
    const uint32_t rowbytes = (uint32_t)X * 2u, planebytes = (uint32_t)umin(YX * 2, 0xFFFFFFFFull);
    float* mytiles = tiles + (size_t)wid * kStages * kPair;
    uint64_t* mybar = bars + wid * kStages;
    if (lane == 0) {
        for (int q = 0; q < kStages; q++) mbar_init(&mybar[q], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const bool use_s = h.shist != nullptr;
    const uint32_t shist_s = use_s ? smem_u32(h.shist) : 0u;
    const uint32_t stride = gridDim.x * kTmaWarps;
    const uint32_t first = blockIdx.x * kTmaWarps + wid;
    // unit = (task, plane pair); the ring runs two units ahead: while pair pr
    // of a task is computed, pair pr + 2 (of this task or the next) loads
    auto issue = [&](uint32_t q, uint32_t bx4, uint32_t by, uint32_t z) {
        mbar_expect_tx(&mybar[q], kPair * 4);
        tma_load_3d(mytiles + q * kPair, &tmap, (int)(bx4 * 32), (int)(by * 8), (int)z, &mybar[q]);
    };
    uint32_t cbx = 0, cby = 0, cbz = 0;   // coordinates of the current task
    if (first < ntask) {
        cbx = first % nbx4;
        const uint32_t t2 = first / nbx4;
        cby = t2 % nby;
        cbz = t2 / nby;
        if (lane == 0) {
            issue(0, cbx, cby, cbz * 8);
            issue(1, cbx, cby, cbz * 8 + 2);
        }
    }
    uint32_t phase = 0;    // bit q: parity of stage q
    uint32_t qc = 0;       // stage of the unit being computed
    bool bad = false;
    // tasks past the first wave are claimed dynamically (the status block's
    // zeroed scratch word), so warps on busier SMs take fewer of them
    unsigned long long* const ctr = &st->pad[2];
    uint32_t nt = 0;
    for (uint32_t task = first; task < ntask; task = nt) {
        const uint32_t bx4 = cbx, by = cby, bz = cbz;
        uint32_t claim = 0;
        if (lane == 0) claim = (uint32_t)atomicAdd(ctr, 1ull);   // consumed at pair 2
        bool has_next = false;
        const uint64_t x = (uint64_t)bx4 * 32 + lane, y0 = (uint64_t)by * 8, z0 = (uint64_t)bz * 8;
        const bool xin = x < X;
        const int ny = (int)umin(8, Y - y0), nz = (int)umin(8, Z - z0);
        const uint64_t base = z0 * YX + y0 * X + x;
        uint16_t* const tb = codes + base;
        const bool full = __all_sync(kFull, xin) && ny == 8 && nz == 8;   // warp-uniform
        int hprev[8];
#pragma unroll
        for (int y = 0; y < 8; y++) hprev[y] = 0;
        bool mark = false;
#pragma unroll 1
        for (uint32_t pr = 0; pr < 4; pr++) {
            if (pr == 2) {   // the next task: its first two pairs load during pairs 2, 3
                nt = stride + __shfl_sync(kFull, claim, 0);
                has_next = nt < ntask;
                if (has_next) {
                    cbx = nt % nbx4;
                    const uint32_t t2 = nt / nbx4;
                    cby = t2 % nby;
                    cbz = t2 / nby;
                }
            }
            if (lane == 0) {
                const uint32_t qn = qc == 0 ? 2 : qc - 1;   // (qc + 2) % 3
                if (pr < 2) issue(qn, bx4, by, bz * 8 + 2 * (pr + 2));
                else if (has_next) issue(qn, cbx, cby, cbz * 8 + 2 * (pr - 2));
            }
            mbar_wait(&mybar[qc], (phase >> qc) & 1u);
            phase ^= 1u << qc;
            const float* tile = mytiles + qc * kPair;
            qc = qc == 2 ? 0 : qc + 1;
            uint16_t* tbz0 = (uint16_t*)((char*)tb + (uint64_t)(2 * pr) * planebytes);
            uint16_t* tbz1 = (uint16_t*)((char*)tbz0 + planebytes);
            const bool zin0 = xin && (int)(2 * pr) < nz, zin1 = xin && (int)(2 * pr + 1) < nz;
            if (full) {
                if (use_s)
                    dq3d_pair<true, true>(tile, lane, xl, rcp, two_eb, hi_lo, hi_span, r, wbase, hb, shist_s, h, hprev,
                                          mark, tbz0, tbz1, rowbytes, zin0, zin1, ny);
                else
                    dq3d_pair<true, false>(tile, lane, xl, rcp, two_eb, hi_lo, hi_span, r, wbase, hb, shist_s, h, hprev,
                                           mark, tbz0, tbz1, rowbytes, zin0, zin1, ny);
            } else {
                if (use_s)
                    dq3d_pair<false, true>(tile, lane, xl, rcp, two_eb, hi_lo, hi_span, r, wbase, hb, shist_s, h, hprev,
                                           mark, tbz0, tbz1, rowbytes, zin0, zin1, ny);
                else
                    dq3d_pair<false, false>(tile, lane, xl, rcp, two_eb, hi_lo, hi_span, r, wbase, hb, shist_s, h,
                                            hprev, mark, tbz0, tbz1, rowbytes, zin0, zin1, ny);
            }
            __syncwarp();   // the stage is refilled two units later
        }
        if (__any_sync(kFull, mark)) {
            dq3d_uncount(codes, base, YX, X, xin, nz, ny, hb, wbase, h);
            dq3d_task_f64<0>(in, base, YX, X, xin, nz, ny, xl, two_eb, r, codes, h, bad);
        }
    }
    if (__any_sync(kFull, bad) && lane == 0) atomicOr(&st->flags, (unsigned long long)F_NONFINITE);
    __syncthreads();
    // merge the lane-private hot bins: warp w sums bins w, w+8, ... over all warps' lanes
    for (uint32_t j = wid; j < kHot; j += kTmaWarps) {
        uint32_t v = 0;
#pragma unroll
        for (int w = 0; w < kTmaWarps; w++) v += hot[(w * kHot + j) * 32 + lane];
        v = __reduce_add_sync(kFull, v);
        if (lane == 0 && v && wbase + j < cap) {
            if (h.shist) atomicAdd(&h.shist[wbase + j], v);
            else if (h.ghist) atomicAdd(&h.ghist[wbase + j], (unsigned long long)v);
        }
    }
    hist_finish(h);
}

// ----------------------------------------------------------------------------
// 2D, block 16x16
// ----------------------------------------------------------------------------
template <int KIND>
__global__ void __launch_bounds__(kThreads, 2) dq2d_kernel(const void* __restrict__ in, uint64_t Y,
                                                           uint64_t X, uint32_t cap, DevStatus* st,
                                                           uint16_t* __restrict__ codes,
                                                           unsigned long long* ghist) {
    using T = typename Raw<KIND>::T;
    extern __shared__ uint32_t smem_hist[];
    HistCtx h;
    hist_init(h, smem_hist, ghist, cap);
    const double two_eb = st->two_eb;
    const double rcp = __drcp_rn(two_eb);
    const int r = (int)(cap >> 1);
    const uint32_t lane = lane_id(), xl = lane & 15;
    const uint64_t nbx2 = ceil_div(ceil_div(X, 16), 2), nby = ceil_div(Y, 16);
    const uint64_t ntask = nbx2 * nby;
    bool bad = false;
    for (uint64_t task = blockIdx.x * (uint64_t)kWarpsPerCta + (threadIdx.x >> 5); task < ntask;
         task += (uint64_t)gridDim.x * kWarpsPerCta) {
        const uint64_t bx2 = task % nbx2, by = task / nbx2;
        const uint64_t x = bx2 * 32 + lane, y0 = by * 16;
        const bool xin = x < X;
        const int ny = (int)umin(16, Y - y0);
        const uint64_t base = y0 * X + x;
        bool use_int = false;
        if (KIND == 0) {
            float raw[16];
            float mx = 0.f;
#pragma unroll
            for (int y = 0; y < 16; y++) {
                float v = 0.f;
                if (xin && y < ny) v = load_raw<0>(in, base + y * X);
                raw[y] = v;
                mx = fmaxf(mx, fabsf(v));
                bad |= !isfinite(v);
            }
            use_int = __all_sync(kFull, !bad && (double)mx / two_eb < kIntBound);
            if (use_int) {
#pragma unroll
                for (int y = 0; y < 16; y++) raw[y] = __int_as_float(prequant_int(raw[y], rcp, two_eb));
                int gprev = 0;
#pragma unroll
                for (int y = 0; y < 16; y++) {
                    int v = __float_as_int(raw[y]);
                    int left = __shfl_up_sync(kFull, v, 1);
                    int g = v - (xl ? left : 0);
                    int delta = g - gprev;
                    gprev = g;
                    if (xin && y < ny) {
                        uint32_t c = code_of_int(delta, r);
                        codes[base + y * X] = (uint16_t)c;
                        hist_add(h, c);
                    }
                }
            }
        }
        if (!use_int) {
            // (y-1,x) + (y,x-1) - (y-1,x-1)   (dualquant.py:123-124)
            double cprev = 0.0;
            for (int y = 0; y < 16; y++) {
                double q = 0.0;
                if (xin && y < ny) {
                    T v = load_raw<KIND>(in, base + y * X);
                    bad |= !isfinite((double)v);
                    q = to_q<KIND>(v, two_eb);
                }
                const double cm = cprev;
                double n_c = __shfl_up_sync(kFull, q, 1);
                double n_cm = __shfl_up_sync(kFull, cm, 1);
                if (!xl) n_c = n_cm = 0.0;
                const double pred = __dsub_rn(__dadd_rn(cm, n_c), n_cm);
                const double delta = __dsub_rn(q, pred);
                cprev = q;
                if (xin && y < ny) {
                    uint32_t c = code_of_f64(delta, r);
                    codes[base + y * X] = (uint16_t)c;
                    hist_add(h, c);
                }
            }
        }
        hist_flush(h);
    }
    if (__any_sync(kFull, bad) && lane == 0) atomicOr(&st->flags, (unsigned long long)F_NONFINITE);
    hist_finish(h);
}

// ----------------------------------------------------------------------------
// 1D, block 32: task = 16 consecutive blocks (512 points)
// ----------------------------------------------------------------------------
template <int KIND>
__global__ void __launch_bounds__(kThreads, 2) dq1d_kernel(const void* __restrict__ in, uint64_t X,
                                                           uint32_t cap, DevStatus* st,
                                                           uint16_t* __restrict__ codes,
                                                           unsigned long long* ghist) {
    using T = typename Raw<KIND>::T;
    extern __shared__ uint32_t smem_hist[];
    HistCtx h;
    hist_init(h, smem_hist, ghist, cap);
    const double two_eb = st->two_eb;
    const double rcp = __drcp_rn(two_eb);
    const int r = (int)(cap >> 1);
    const uint32_t lane = lane_id();
    const uint64_t ntask = ceil_div(X, 512);
    bool bad = false;
    for (uint64_t task = blockIdx.x * (uint64_t)kWarpsPerCta + (threadIdx.x >> 5); task < ntask;
         task += (uint64_t)gridDim.x * kWarpsPerCta) {
        const uint64_t base = task * 512 + lane;
        bool use_int = false;
        if (KIND == 0) {
            float raw[16];
            float mx = 0.f;
#pragma unroll
            for (int j = 0; j < 16; j++) {
                float v = 0.f;
                if (base + j * 32 < X) v = load_raw<0>(in, base + j * 32);
                raw[j] = v;
                mx = fmaxf(mx, fabsf(v));
                bad |= !isfinite(v);
            }
            use_int = __all_sync(kFull, !bad && (double)mx / two_eb < kIntBound);
            if (use_int) {
#pragma unroll
                for (int j = 0; j < 16; j++) raw[j] = __int_as_float(prequant_int(raw[j], rcp, two_eb));
#pragma unroll
                for (int j = 0; j < 16; j++) {
                    int v = __float_as_int(raw[j]);
                    int left = __shfl_up_sync(kFull, v, 1);
                    int delta = v - (lane ? left : 0);
                    if (base + j * 32 < X) {
                        uint32_t c = code_of_int(delta, r);
                        codes[base + j * 32] = (uint16_t)c;
                        hist_add(h, c);
                    }
                }
            }
        }
        if (!use_int) {
            for (int j = 0; j < 16; j++) {
                const uint64_t i = base + j * 32;
                double q = 0.0;
                if (i < X) {
                    T v = load_raw<KIND>(in, i);
                    bad |= !isfinite((double)v);
                    q = to_q<KIND>(v, two_eb);
                }
                double n_c = __shfl_up_sync(kFull, q, 1);
                if (!lane) n_c = 0.0;
                const double delta = __dsub_rn(q, n_c);
                if (i < X) {
                    uint32_t c = code_of_f64(delta, r);
                    codes[i] = (uint16_t)c;
                    hist_add(h, c);
                }
            }
        }
        hist_flush(h);
    }
    if (__any_sync(kFull, bad) && lane == 0) atomicOr(&st->flags, (unsigned long long)F_NONFINITE);
    hist_finish(h);
}

// ----------------------------------------------------------------------------
// 1D, block 32, fp32, whole 1024-point tasks.  Lane l holds points 4l..4l+3 of
// each of the task's 8 rows of 128 (float4 loads, 8 in flight per lane; one
// uint2 store of 4 codes), a block spans 8 lanes.  Prequantization is the
// fixed-point FMA of dq3d_tma_kernel (bias kFixK cancels in the differences;
// the left neighbour of a block's first point is the bias itself, i.e. the
// zero pad of dualquant.py:81-86), with the same exact tie-neighbourhood
// redo.  A task holding any |v / 2eb| >= 2^27 - 2048 (or a non-finite value)
// is computed in fp64 with exact division instead (dualquant.py:76-77, 1D
// predictor d[a-1]).  Histogram: lane-private hot bins + CTA bins (one shared
// reduction per point).
// ----------------------------------------------------------------------------
constexpr uint32_t kVecTask = 1024;

template <bool SH>
__device__ __forceinline__ void dq1d_count(uint32_t c, uint32_t wbase, uint32_t hb, uint32_t shist_s,
                                           HistCtx& h) {
    if (SH) {
        const bool hot = c - wbase < kHot;
        const uint32_t addr = c * (hot ? 128u : 4u) + (hot ? hb : shist_s);
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
    } else {
        hot_add(hb, c, wbase, h, 1);
    }
}

// exact fp64 task (dualquant.py:76-77, predictor d[a-1]), reloading its values
template <bool SH>
__device__ __noinline__ void dq1d_task_f64(const float4* __restrict__ src, uint2* __restrict__ dst,
                                           uint32_t lane, double two_eb, int r, uint32_t wbase,
                                           uint32_t hb, uint32_t shist_s, HistCtx h, bool& bad,
                                           double* __restrict__ hd) {
    const bool lead = (lane & 7) == 0;
    for (int j = 0; j < 8; j++) {
        const float4 w = __ldg(src + 32 * j);
        const float e[4] = {w.x, w.y, w.z, w.w};
        double d[4];
#pragma unroll
        for (int c = 0; c < 4; c++) {
            bad |= !isfinite(e[c]);
            d[c] = prequant((double)e[c], two_eb);
        }
        double left = __shfl_up_sync(kFull, d[3], 1);
        if (lead) left = 0.0;
        uint32_t cc[4];
#pragma unroll
        for (int c = 0; c < 4; c++) {
            cc[c] = code_of_f64(__dsub_rn(d[c], c ? d[c - 1] : left), r);
            dq1d_count<SH>(cc[c], wbase, hb, shist_s, h);
        }
        if (hd && lead && cc[0] == 0) hd[(32 * j + lane) >> 3] = d[0];
        dst[32 * j] = make_uint2(cc[0] | (cc[1] << 16), cc[2] | (cc[3] << 16));
    }
}

template <bool SH>
__global__ void __launch_bounds__(kThreads, 2) dq1d_vec_kernel(const float* __restrict__ in, uint64_t ntask,
                                                               uint32_t cap, DevStatus* st,
                                                               uint16_t* __restrict__ codes,
                                                               unsigned long long* ghist,
                                                               double* __restrict__ heads) {
    extern __shared__ __align__(16) uint32_t dsm1[];
    uint32_t* hot = dsm1;   // [warp][kHot][32]
    for (uint32_t i = threadIdx.x; i < kWarpsPerCta * kHot * 32; i += blockDim.x) hot[i] = 0;
    HistCtx h;
    hist_init(h, hot + kWarpsPerCta * kHot * 32, ghist, cap);   // (syncs)
    const double two_eb = st->two_eb;
    const double rcp = __drcp_rn(two_eb);
    const uint32_t hi_lo = (uint32_t)__double2hiint(kFixC - kFixBound) + 1u;
    const uint32_t hi_span = (uint32_t)__double2hiint(kFixC + kFixBound) - hi_lo;
    const int r = (int)(cap >> 1);
    const uint32_t wbase = cap >= 2 * kHot ? (uint32_t)r - kHot / 2 : 0u;
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    const uint32_t hb = smem_u32(hot + wid * kHot * 32 + lane) - wbase * 128u;
    const uint32_t shist_s = SH ? smem_u32(h.shist) : 0u;
    const bool lead = (lane & 7) == 0;   // first lane of a 32-point block
    bool bad = false;
    for (uint64_t task = blockIdx.x * (uint64_t)kWarpsPerCta + wid; task < ntask;
         task += (uint64_t)gridDim.x * kWarpsPerCta) {
        const float4* src = reinterpret_cast<const float4*>(in + task * kVecTask) + lane;
        uint2* dst = reinterpret_cast<uint2*>(codes + task * kVecTask) + lane;
        float4 v[8];
#pragma unroll
        for (int j = 0; j < 8; j++) v[j] = __ldcs(src + 32 * j);
        int q[8][4];
        bool amb = false, mark = false;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const float e[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const double R = __fma_rn((double)e[c], rcp, kFixC);
                const uint32_t lo = (uint32_t)__double2loint(R), hi = (uint32_t)__double2hiint(R);
                amb |= (lo & 0x3FFFFCu) == 0u;
                mark |= (hi - hi_lo) >= hi_span;
                q[j][c] = (int)__funnelshift_r(lo, hi, 22);
            }
        }
        double* hd = heads ? heads + task * (kVecTask / 32) : nullptr;   // this task's 32 block heads
        if (__any_sync(kFull, mark)) {   // rare: huge magnitudes or non-finite values
            dq1d_task_f64<SH>(src, dst, lane, two_eb, r, wbase, hb, shist_s, h, bad, hd);
            continue;
        }
        if (__any_sync(kFull, amb)) {   // rare: exact division near a rounding tie
#pragma unroll 1
            for (int j = 0; j < 8; j++) {
                const float4 w = __ldg(src + 32 * j);
                const float e[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const double R = __fma_rn((double)e[c], rcp, kFixC);
                    if (((uint32_t)__double2loint(R) & 0x3FFFFCu) == 0u) {
                        const int m = (int)floor(__dadd_rn(fabs(__ddiv_rn((double)e[c], two_eb)), 0.5));
                        const int qq = (e[c] < 0.f ? -m : m) + kFixK;
#pragma unroll
                        for (int jj = 0; jj < 8; jj++)
                            if (jj == j) q[jj][c] = qq;
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 8; j++) {
            int left = __shfl_up_sync(kFull, q[j][3], 1);
            if (lead) left = kFixK;
            uint32_t cc[4];
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const uint32_t uu = (uint32_t)(q[j][c] - (c ? q[j][c - 1] : left) + r);
                cc[c] = (uu - 1u) < (uint32_t)(2 * r - 1) ? uu : 0u;   // -r < delta < r
                dq1d_count<SH>(cc[c], wbase, hb, shist_s, h);
            }
            // an outlier block head (|q| >= r >= 2, so never -0.0): its exact prequantized value
            if (hd && lead && cc[0] == 0) hd[(32 * j + lane) >> 3] = (double)(q[j][0] - kFixK);
            dst[32 * j] = make_uint2(cc[0] | (cc[1] << 16), cc[2] | (cc[3] << 16));
        }
    }
    if (__any_sync(kFull, bad) && lane == 0) atomicOr(&st->flags, (unsigned long long)F_NONFINITE);
    __syncthreads();
    for (uint32_t j = wid; j < kHot; j += kWarpsPerCta) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < kWarpsPerCta; w++) s += hot[(w * kHot + j) * 32 + lane];
        s = __reduce_add_sync(kFull, s);
        if (lane == 0 && s && wbase + j < cap) {
            if (h.shist) atomicAdd(&h.shist[wbase + j], s);
            else if (h.ghist) atomicAdd(&h.ghist[wbase + j], (unsigned long long)s);
        }
    }
    hist_finish(h);
}

// ----------------------------------------------------------------------------
// 2D, block 16x16, fp32, row pitch a multiple of 4 floats.  A task is 16 rows
// x 128 columns (8 blocks side by side); lane l holds columns 4l..4l+3 of
// each row (float4 loads, uint2 code stores), a block spans 4 lanes.  The
// task's 64 prequantized values per lane (fixed-point FMA as in
// dq3d_tma_kernel) stay in registers; D_x by one shuffle per row, D_y against
// the previous row.  A task holding any |v / 2eb| >= 2^27 - 2048 (or a
// non-finite value) is computed in fp64 with exact division in the
// reference's term order (dualquant.py:123-124); values near a rounding tie
// are redone with exact division.
// ----------------------------------------------------------------------------
template <bool SH>
__device__ __noinline__ void dq2d_task_f64(const float* __restrict__ in, uint16_t* __restrict__ codes,
                                           uint64_t X, uint64_t y0, int ny, uint64_t x0, bool xin,
                                           uint32_t lane, double two_eb, int r, uint32_t wbase, uint32_t hb,
                                           uint32_t shist_s, HistCtx h, bool& bad) {
    const bool lead = (lane & 3) == 0;
    double prev[4] = {0.0, 0.0, 0.0, 0.0};
    for (int y = 0; y < 16; y++) {
        const bool row = xin && y < ny;
        float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row) w = __ldg(reinterpret_cast<const float4*>(in + (y0 + y) * X + x0));
        const float e[4] = {w.x, w.y, w.z, w.w};
        double q[4];
#pragma unroll
        for (int c = 0; c < 4; c++) {
            bad |= row && !isfinite(e[c]);
            q[c] = row ? prequant((double)e[c], two_eb) : 0.0;
        }
        double lq = __shfl_up_sync(kFull, q[3], 1), lp = __shfl_up_sync(kFull, prev[3], 1);
        if (lead) lq = lp = 0.0;
        uint32_t cc[4];
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const double nc = c ? q[c - 1] : lq, ncm = c ? prev[c - 1] : lp;
            const double pred = __dsub_rn(__dadd_rn(prev[c], nc), ncm);
            cc[c] = code_of_f64(__dsub_rn(q[c], pred), r);
        }
#pragma unroll
        for (int c = 0; c < 4; c++) prev[c] = q[c];
        if (row) {
#pragma unroll
            for (int c = 0; c < 4; c++) dq1d_count<SH>(cc[c], wbase, hb, shist_s, h);
            *reinterpret_cast<uint2*>(codes + (y0 + y) * X + x0) =
                make_uint2(cc[0] | (cc[1] << 16), cc[2] | (cc[3] << 16));
        }
    }
}

template <bool SH>
__global__ void __launch_bounds__(kThreads, 2) dq2d_vec_kernel(const float* __restrict__ in, uint64_t Y,
                                                               uint64_t X, uint32_t cap, DevStatus* st,
                                                               uint16_t* __restrict__ codes,
                                                               unsigned long long* ghist) {
    extern __shared__ __align__(16) uint32_t dsm2[];
    uint32_t* hot = dsm2;   // [warp][kHot][32]
    for (uint32_t i = threadIdx.x; i < kWarpsPerCta * kHot * 32; i += blockDim.x) hot[i] = 0;
    HistCtx h;
    hist_init(h, hot + kWarpsPerCta * kHot * 32, ghist, cap);   // (syncs)
    const double two_eb = st->two_eb;
    const double rcp = __drcp_rn(two_eb);
    const uint32_t hi_lo = (uint32_t)__double2hiint(kFixC - kFixBound) + 1u;
    const uint32_t hi_span = (uint32_t)__double2hiint(kFixC + kFixBound) - hi_lo;
    const int r = (int)(cap >> 1);
    const uint32_t wbase = cap >= 2 * kHot ? (uint32_t)r - kHot / 2 : 0u;
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    const uint32_t hb = smem_u32(hot + wid * kHot * 32 + lane) - wbase * 128u;
    const uint32_t shist_s = SH ? smem_u32(h.shist) : 0u;
    const bool lead = (lane & 3) == 0;   // first lane of a 16-column block
    const uint64_t ntx = ceil_div(X, 128), nty = ceil_div(Y, 16), ntask = ntx * nty;
    bool bad = false;
    for (uint64_t task = blockIdx.x * (uint64_t)kWarpsPerCta + wid; task < ntask;
         task += (uint64_t)gridDim.x * kWarpsPerCta) {
        const uint64_t tx = task % ntx, ty = task / ntx;
        const uint64_t x0 = tx * 128 + lane * 4, y0 = ty * 16;
        const bool xin = x0 < X;
        const int ny = (int)umin(16, Y - y0);
        const float* src = in + y0 * X + x0;
        int q[16][4];
        bool amb = false, mark = false;
#pragma unroll
        for (int hh = 0; hh < 4; hh++) {
            float4 v[4];
#pragma unroll
            for (int y = 0; y < 4; y++) {
                v[y] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (xin && hh * 4 + y < ny) v[y] = __ldcs(reinterpret_cast<const float4*>(src + (hh * 4 + y) * X));
            }
#pragma unroll
            for (int y = 0; y < 4; y++) {
                const float e[4] = {v[y].x, v[y].y, v[y].z, v[y].w};
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const double R = __fma_rn((double)e[c], rcp, kFixC);
                    const uint32_t lo = (uint32_t)__double2loint(R), hi = (uint32_t)__double2hiint(R);
                    amb |= (lo & 0x3FFFFCu) == 0u;
                    mark |= (hi - hi_lo) >= hi_span;
                    q[hh * 4 + y][c] = (int)__funnelshift_r(lo, hi, 22);
                }
            }
        }
        if (__any_sync(kFull, mark)) {   // rare: huge magnitudes or non-finite values
            dq2d_task_f64<SH>(in, codes, X, y0, ny, x0, xin, lane, two_eb, r, wbase, hb, shist_s, h, bad);
            continue;
        }
        if (__any_sync(kFull, amb)) {   // rare: exact division near a rounding tie
#pragma unroll
            for (int y = 0; y < 16; y++) {
                if (!(xin && y < ny)) continue;
                const float4 w = __ldg(reinterpret_cast<const float4*>(src + y * X));
                const float e[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const double R = __fma_rn((double)e[c], rcp, kFixC);
                    if (((uint32_t)__double2loint(R) & 0x3FFFFCu) == 0u) {
                        const int m = (int)floor(__dadd_rn(fabs(__ddiv_rn((double)e[c], two_eb)), 0.5));
                        q[y][c] = (e[c] < 0.f ? -m : m) + kFixK;
                    }
                }
            }
        }
        int gprev[4] = {0, 0, 0, 0};
#pragma unroll
        for (int y = 0; y < 16; y++) {
            int left = __shfl_up_sync(kFull, q[y][3], 1);
            if (lead) left = kFixK;
            uint32_t cc[4];
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const int g = q[y][c] - (c ? q[y][c - 1] : left);
                const uint32_t uu = (uint32_t)(g - gprev[c] + r);
                gprev[c] = g;
                cc[c] = (uu - 1u) < (uint32_t)(2 * r - 1) ? uu : 0u;   // -r < delta < r
            }
            if (xin && y < ny) {
#pragma unroll
                for (int c = 0; c < 4; c++) dq1d_count<SH>(cc[c], wbase, hb, shist_s, h);
                *reinterpret_cast<uint2*>(codes + (y0 + y) * X + x0) =
                    make_uint2(cc[0] | (cc[1] << 16), cc[2] | (cc[3] << 16));
            }
        }
    }
    if (__any_sync(kFull, bad) && lane == 0) atomicOr(&st->flags, (unsigned long long)F_NONFINITE);
    __syncthreads();
    for (uint32_t j = wid; j < kHot; j += kWarpsPerCta) {
        uint32_t sum = 0;
#pragma unroll
        for (int w = 0; w < kWarpsPerCta; w++) sum += hot[(w * kHot + j) * 32 + lane];
        sum = __reduce_add_sync(kFull, sum);
        if (lane == 0 && sum && wbase + j < cap) {
            if (h.shist) atomicAdd(&h.shist[wbase + j], sum);
            else if (h.ghist) atomicAdd(&h.ghist[wbase + j], (unsigned long long)sum);
        }
    }
    hist_finish(h);
}

// ----------------------------------------------------------------------------
// Generic block shapes: one thread per point, fp64 reference order.
// ----------------------------------------------------------------------------
struct Geo {
    int nd;
    uint64_t dims[3];
    uint32_t block[3];
    uint64_t stride[3];
    uint64_t nblk[3];
};

template <int KIND>
__global__ void __launch_bounds__(kThreads) dq_generic_kernel(const void* __restrict__ in, Geo g,
                                                              uint64_t n, uint32_t cap,
                                                              DevStatus* st,
                                                              uint16_t* __restrict__ codes,
                                                              unsigned long long* ghist) {
    extern __shared__ uint32_t smem_hist[];
    HistCtx h;
    hist_init(h, smem_hist, ghist, cap);
    const double two_eb = st->two_eb;
    const double rcp = __drcp_rn(two_eb);
    const int r = (int)(cap >> 1);
    bool bad = false;
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t ntot = ceil_div(n, 32) * 32;   // keep whole warps alive for the flushes
    uint32_t cnt = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ntot; i += stride) {
        if (i < n) {
            uint64_t c[3] = {0, 0, 0}, rem = i;
            bool lead[3] = {true, true, true};
            for (int a = 0; a < g.nd; a++) {
                c[a] = rem / g.stride[a];
                rem -= c[a] * g.stride[a];
                lead[a] = (c[a] % g.block[a]) == 0;   // neighbour at -1 is padding
            }
            auto val = [&](int da, int db, int dc) -> double {
                int dd[3] = {da, db, dc};
                uint64_t j = i;
                for (int a = 0; a < g.nd; a++) {
                    if (dd[a]) {
                        if (lead[a]) return 0.0;
                        j -= g.stride[a];
                    }
                }
                return load_q<KIND>(in, j, two_eb, bad);
            };
            double q = val(0, 0, 0);
            double pred;
            if (g.nd == 1) {
                pred = val(1, 0, 0);
            } else if (g.nd == 2) {
                pred = __dsub_rn(__dadd_rn(val(1, 0, 0), val(0, 1, 0)), val(1, 1, 0));
            } else {
                pred = __dadd_rn(val(1, 0, 0), val(0, 1, 0));
                pred = __dadd_rn(pred, val(0, 0, 1));
                pred = __dsub_rn(pred, val(1, 1, 0));
                pred = __dsub_rn(pred, val(1, 0, 1));
                pred = __dsub_rn(pred, val(0, 1, 1));
                pred = __dadd_rn(pred, val(1, 1, 1));
            }
            uint32_t code = code_of_f64(__dsub_rn(q, pred), r);
            codes[i] = (uint16_t)code;
            hist_add(h, code);
        }
        if (++cnt == 200) {   // 8-bit packed counters: flush well before 255
            hist_flush(h);
            cnt = 0;
        }
    }
    hist_flush(h);
    if (__any_sync(kFull, bad) && lane_id() == 0) atomicOr(&st->flags, (unsigned long long)F_NONFINITE);
    hist_finish(h);
}

// ----------------------------------------------------------------------------
// Generic block shapes, one thread per block (blocks of <= kBlkMaxSlots plane +
// row slots): the block is walked in raster order; the prequantized values
// of the previous row (R[x]) and of the previous plane (P[y][x]) sit in the
// thread's shared-memory slots ([slot][thread], conflict-free), the x - 1
// neighbours in registers, so every point is prequantized once and its
// Lorenzo prediction is the reference's fp64 expression in the reference's
// term order (dualquant.py:81-129; exactly dq_generic_kernel's arithmetic).
// P[y-1][x] is overwritten with the current plane's row y-1 as soon as row y
// has read it, and the last row moves in at the end of the plane.
// ----------------------------------------------------------------------------
constexpr uint32_t kBlkMaxSlots = 512;   // per-thread fp64 slots (4 KB)

__host__ __device__ __forceinline__ uint32_t blk_slots(int nd, const uint32_t* block) {
    const uint32_t bx = block[nd - 1], by = nd >= 2 ? block[nd - 2] : 1;
    return (nd == 3 ? bx * by : 0) + (nd >= 2 ? bx : 0);
}

// per-thread flush of the packed window counters (no warp synchronisation:
// threads of a warp walk blocks of different sizes)
__device__ __forceinline__ void hist_flush_thread(HistCtx& h) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
        const uint32_t c = (uint32_t)(((k < 8) ? (h.lo >> (8 * k)) : (h.hi >> (8 * (k - 8)))) & 0xFF);
        if (c) {
            if (h.shist) atomicAdd(&h.shist[h.wbase + k], c);
            else if (h.ghist) atomicAdd(&h.ghist[h.wbase + k], (unsigned long long)c);
        }
    }
    h.lo = h.hi = 0;
}

template <int KIND, int ND>
__global__ void __launch_bounds__(64) dq_blocks_kernel(const void* __restrict__ in, Geo g, uint32_t cap,
                                                       uint32_t hist_bytes, DevStatus* st,
                                                       uint16_t* __restrict__ codes, unsigned long long* ghist) {
    extern __shared__ __align__(128) unsigned char dsm[];
    HistCtx h;
    hist_init(h, reinterpret_cast<uint32_t*>(dsm), ghist, cap);
    const uint32_t T = blockDim.x, tid = threadIdx.x;
    double* buf = reinterpret_cast<double*>(dsm + hist_bytes) + tid;   // slot s at buf[s * T]
    constexpr int nd = ND;
    const uint32_t bx = g.block[nd - 1], by = nd >= 2 ? g.block[nd - 2] : 1;
    double* P = buf;                                          // [by][bx] (3D)
    double* R = buf + (size_t)(nd == 3 ? bx * by : 0) * T;    // [bx] (2D, 3D)
    const uint64_t nbx = g.nblk[nd - 1], nby = nd >= 2 ? g.nblk[nd - 2] : 1;
    const uint64_t nblocks = g.nblk[0] * g.nblk[1] * g.nblk[2];
    const uint64_t sy = nd >= 2 ? g.stride[nd - 2] : 0, sz = nd == 3 ? g.stride[0] : 0;
    const uint64_t X = g.dims[nd - 1], Y = nd >= 2 ? g.dims[nd - 2] : 1, Z = nd == 3 ? g.dims[0] : 1;
    const uint32_t bz = nd == 3 ? g.block[0] : 1;
    const double two_eb = st->two_eb;
    const double rcp = __drcp_rn(two_eb);
    const int r = (int)(cap >> 1);
    bool bad = false;
    uint32_t cnt = 0;
    for (uint64_t b = blockIdx.x * (uint64_t)T + tid; b < nblocks; b += (uint64_t)gridDim.x * T) {
        const uint64_t cx = b % nbx, t2 = b / nbx, cy = t2 % nby, cz = t2 / nby;
        const uint32_t nx = (uint32_t)umin(bx, X - cx * bx), ny = (uint32_t)umin(by, Y - cy * by),
                       nz = (uint32_t)umin(bz, Z - cz * bz);
        const uint64_t base = cz * bz * sz + cy * by * sy + cx * bx;
        for (uint32_t z = 0; z < nz; z++) {
            for (uint32_t y = 0; y < ny; y++) {
                double a = 0.0, e = 0.0, f = 0.0, gq = 0.0;   // (x-1) neighbours: own row, row y-1, plane z-1, both
                const uint64_t rb = base + z * sz + y * sy;
                for (uint32_t x = 0; x < nx; x++) {
                    const double q = load_q_fast<KIND>(in, rb + x, two_eb, rcp, bad);
                    const double bb = (nd >= 2 && y > 0) ? R[(size_t)x * T] : 0.0;
                    const double cc = (nd == 3 && z > 0) ? P[(size_t)(y * bx + x) * T] : 0.0;
                    const double dd = (nd == 3 && z > 0 && y > 0) ? P[(size_t)((y - 1) * bx + x) * T] : 0.0;
                    double pred;
                    if (nd == 1) {
                        pred = a;
                    } else if (nd == 2) {
                        pred = __dsub_rn(__dadd_rn(bb, a), e);
                    } else {
                        pred = __dadd_rn(cc, bb);
                        pred = __dadd_rn(pred, a);
                        pred = __dsub_rn(pred, dd);
                        pred = __dsub_rn(pred, f);
                        pred = __dsub_rn(pred, e);
                        pred = __dadd_rn(pred, gq);
                    }
                    const uint32_t code = code_of_f64(__dsub_rn(q, pred), r);
                    codes[rb + x] = (uint16_t)code;
                    hist_add(h, code);
                    if (++cnt == 200) {   // 8-bit packed counters
                        hist_flush_thread(h);
                        cnt = 0;
                    }
                    if (nd == 3 && y > 0) P[(size_t)((y - 1) * bx + x) * T] = bb;   // plane z, row y-1
                    if (nd >= 2) R[(size_t)x * T] = q;
                    a = q;
                    e = bb;
                    f = cc;
                    gq = dd;
                }
            }
            if (nd == 3)
                for (uint32_t x = 0; x < nx; x++) P[(size_t)((ny - 1) * bx + x) * T] = R[(size_t)x * T];
        }
    }
    hist_flush_thread(h);
    if (bad) atomicOr(&st->flags, (unsigned long long)F_NONFINITE);
    hist_finish(h);
}

// prequantized value of an already loaded input element (load_q_fast without the load)
template <int KIND>
__device__ __forceinline__ double q_of(typename std::conditional<KIND == 0, float, double>::type v, double two_eb,
                                       double rcp, bool& bad) {
    bad |= !isfinite(v);
    if (KIND == 2) return v;
    if (KIND == 0) {
        const double y = __dmul_rn((double)v, rcp);
        const double ay = fabs(y);
        if (ay < 134217728.0) {
            const double t = __dadd_rn(ay, 0.5);
            const double fl = floor(t);
            const double fr = __dsub_rn(t, fl);
            if (fr >= 2.384185791015625e-07 && fr <= 1.0 - 2.384185791015625e-07) return copysign(fl, y);
        }
    }
    return prequant((double)v, two_eb);
}

// Generic block shapes, one thread per block-row segment (3D/2D: the x-extent
// of one block in one row; 1D: one point): every neighbour the reference's
// prediction reads is prequantized again by this thread (x-1 values carried
// along the row), so each segment is independent -- millions of threads and
// coalesced row reads where dq_blocks_kernel has one sequential thread per
// block.  Same fp64 expression and term order (dualquant.py:81-129).
template <int KIND, int ND>
__global__ void __launch_bounds__(256) dq_rows_kernel(const void* __restrict__ in, Geo g, uint64_t nitems,
                                                      uint32_t cap, DevStatus* st, uint16_t* __restrict__ codes,
                                                      unsigned long long* ghist) {
    extern __shared__ __align__(128) unsigned char rsm[];
    HistCtx h;
    hist_init(h, reinterpret_cast<uint32_t*>(rsm), ghist, cap);
    constexpr int nd = ND;
    const uint32_t bx = g.block[nd - 1], by = nd >= 2 ? g.block[nd - 2] : 1, bz = nd == 3 ? g.block[0] : 1;
    const uint64_t X = g.dims[nd - 1], Y = nd >= 2 ? g.dims[nd - 2] : 1;
    const uint64_t nbx = g.nblk[nd - 1];
    const uint64_t sy = nd >= 2 ? g.stride[nd - 2] : 0, sz = nd == 3 ? g.stride[0] : 0;
    const double two_eb = st->two_eb;
    const double rcp = __drcp_rn(two_eb);
    const int r = (int)(cap >> 1);
    bool bad = false;
    uint32_t cnt = 0;
    auto emit = [&](uint64_t i, double delta) {
        const uint32_t code = code_of_f64(delta, r);
        codes[i] = (uint16_t)code;
        hist_add(h, code);
        if (++cnt == 200) {   // 8-bit packed counters
            hist_flush_thread(h);
            cnt = 0;
        }
    };
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    if (nd == 1) {   // warp per 512-point task, lane = point: the left neighbour is the lane to the left's q
        using raw_t = typename std::conditional<KIND == 0, float, double>::type;
        constexpr int kG = 16;   // 32-point steps per task, loaded together
        const uint32_t lane = threadIdx.x & 31;
        const uint64_t nw = stride >> 5, ntask = ceil_div(nitems, 32 * kG);
        const uint32_t step = 32 % bx;
        for (uint64_t t = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; t < ntask; t += nw) {
            const uint64_t i0 = t * 32 * kG;
            raw_t v[kG];
#pragma unroll
            for (int k = 0; k < kG; k++) {
                const uint64_t i = i0 + 32 * k + lane;
                v[k] = i < nitems ? __ldg((const raw_t*)in + i) : (raw_t)0;
            }
            // the point before the task (lane 0's left neighbour at step 0)
            double carry = (lane == 0 && i0 > 0 && (i0 % bx) != 0) ? load_q_fast<KIND>(in, i0 - 1, two_eb, rcp, bad) : 0.0;
            uint32_t pos = (uint32_t)((i0 + lane) % bx);
#pragma unroll
            for (int k = 0; k < kG; k++) {
                const uint64_t i = i0 + 32 * k + lane;
                const bool in_range = i < nitems;
                const double q = in_range ? q_of<KIND>(v[k], two_eb, rcp, bad) : 0.0;
                double a = __shfl_up_sync(kFull, q, 1);
                if (lane == 0) a = carry;
                carry = __shfl_sync(kFull, q, 31);
                if (pos == 0) a = 0.0;
                if (in_range) emit(i, __dsub_rn(q, a));
                pos += step;
                if (pos >= bx) pos -= bx;
            }
        }
    }
    for (uint64_t it = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; nd > 1 && it < nitems; it += stride) {
        const uint64_t cx = it % nbx, row = it / nbx;
        const uint64_t y = row % Y, z = row / Y;
        const bool hy = (y % by) != 0, hz = nd == 3 && (z % bz) != 0;   // neighbours inside the block
        const uint64_t x0 = cx * bx;
        const uint32_t nx = (uint32_t)umin(bx, X - x0);
        const uint64_t rb = z * sz + y * sy + x0;
        double a = 0.0, e = 0.0, f = 0.0, gq = 0.0;   // (x-1): own row, row y-1, plane z-1, both
        for (uint32_t x = 0; x < nx; x++) {
            const uint64_t i = rb + x;
            const double q = load_q_fast<KIND>(in, i, two_eb, rcp, bad);
            const double bb = hy ? load_q_fast<KIND>(in, i - sy, two_eb, rcp, bad) : 0.0;
            double pred;
            if (nd == 2) {
                pred = __dsub_rn(__dadd_rn(bb, a), e);
            } else {
                const double cc = hz ? load_q_fast<KIND>(in, i - sz, two_eb, rcp, bad) : 0.0;
                const double dd = (hy && hz) ? load_q_fast<KIND>(in, i - sz - sy, two_eb, rcp, bad) : 0.0;
                pred = __dadd_rn(cc, bb);
                pred = __dadd_rn(pred, a);
                pred = __dsub_rn(pred, dd);
                pred = __dsub_rn(pred, f);
                pred = __dsub_rn(pred, e);
                pred = __dadd_rn(pred, gq);
                f = cc;
                gq = dd;
            }
            emit(i, __dsub_rn(q, pred));
            a = q;
            e = bb;
        }
    }
    hist_flush_thread(h);
    if (bad) atomicOr(&st->flags, (unsigned long long)F_NONFINITE);
    hist_finish(h);
}

// dq_strip_kernel's Lorenzo prediction of the point with prequantized value q
// (T = int when every value is below 2^27, else double): row y-1 / plane z-1
// from the lane-private slots (which it then updates), x-1 from the lane to the
// left or the carried lane 31 of the previous segment.  Term order of
// dualquant.py:81-129.
template <typename T, bool ONE>
__device__ __forceinline__ T strip_pred(int nd, T q, double* R, double* D, double* P, uint32_t s, uint32_t y,
                                        uint32_t z, uint32_t steps, bool seg0, uint32_t lane, T& cq, T& cb, T& ccq,
                                        T& cdq) {
    T* Rs = reinterpret_cast<T*>(R + s * 32);
    const T bb = y > 0 ? *Rs : T(0);
    T cc = T(0), dd = T(0);
    if (nd == 3) {
        T* pp = reinterpret_cast<T*>(P + (size_t)(y * steps + s) * 32);
        T* Ds = reinterpret_cast<T*>(D + s * 32);
        if (z > 0) {
            cc = *pp;
            dd = y > 0 ? *Ds : T(0);
        }
        *Ds = cc;   // row y of plane z-1, for row y+1
        *pp = q;
    }
    *Rs = q;
    T a = __shfl_up_sync(kFull, q, 1), e = __shfl_up_sync(kFull, bb, 1), f = T(0), gq = T(0);
    if (nd == 3) {
        f = __shfl_up_sync(kFull, cc, 1);
        gq = __shfl_up_sync(kFull, dd, 1);
    }
    if (!ONE) {
        if (lane == 0) { a = cq; e = cb; f = ccq; gq = cdq; }
        cq = __shfl_sync(kFull, q, 31);
        cb = __shfl_sync(kFull, bb, 31);
        if (nd == 3) {
            ccq = __shfl_sync(kFull, cc, 31);
            cdq = __shfl_sync(kFull, dd, 31);
        }
    }
    if (ONE ? seg0 : (seg0 && s == 0)) a = e = f = gq = T(0);
    if constexpr (sizeof(T) == 4) {
        return nd == 2 ? bb + a - e : cc + bb + a - dd - f - e + gq;
    } else {
        if (nd == 2) return __dsub_rn(__dadd_rn(bb, a), e);
        T p = __dadd_rn(cc, bb);
        p = __dadd_rn(p, a);
        p = __dsub_rn(p, dd);
        p = __dsub_rn(p, f);
        p = __dsub_rn(p, e);
        return __dadd_rn(p, gq);
    }
}

constexpr int kStripPf = 16;  // strip-kernel rows in flight (cp.async ring slots) per warp

// 2D / 3D generic block shapes, warp per strip of block columns (the layout
// of rq_rows_kernel): 32 / bx whole blocks side by side when bx <= 32 (ONE),
// one block in `steps` 32-lane segments otherwise, over nyb block rows;
// lane = column, rows in sequence.  Each point is loaded and prequantized
// once: the x-1 neighbours come from the lane to the left (shuffle; the
// previous segment's lane 31 across segments), row y-1 and plane z-1 from
// lane-private shared-memory slots.  Same fp64 expression and term order as
// dq_blocks_kernel (dualquant.py:81-129).
template <int KIND, bool ONE, int ND>
__global__ void __launch_bounds__(256) dq_strip_kernel(const void* __restrict__ in, Geo g, uint32_t W,
                                                       uint32_t steps, uint32_t nyb, uint32_t cap,
                                                       uint32_t hist_bytes, DevStatus* st,
                                                       uint16_t* __restrict__ codes,
                                                       unsigned long long* ghist) {
    using raw_t = typename std::conditional<KIND == 0, float, double>::type;
    extern __shared__ __align__(128) unsigned char ssm[];
    HistCtx h;
    hist_init(h, reinterpret_cast<uint32_t*>(ssm), ghist, cap);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int nd = ND;   // 2 or 3 (template: no per-point dimension branches)
    const uint32_t bx = g.block[nd - 1], by = g.block[nd - 2], bz = nd == 3 ? g.block[0] : 1;
    const uint32_t per_warp = steps * (nd == 3 ? 2 + by : 1) * 32;
    double* R = reinterpret_cast<double*>(ssm + hist_bytes) + warp * per_warp + lane;   // [steps]: q of row y-1
    double* D = R + steps * 32;                 // [steps]: q of row y-1 in plane z-1 (3D)
    double* P = D + steps * 32;                 // [by][steps]: q of plane z-1 (3D)
    const raw_t* ring = reinterpret_cast<const raw_t*>(ssm + hist_bytes + (size_t)(blockDim.x >> 5) * per_warp * sizeof(double)) +
                        warp * kStripPf * 32 + lane;   // [kStripPf][32] loads in flight
    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
    const uint64_t X = g.dims[nd - 1], Y = g.dims[nd - 2], Z = nd == 3 ? g.dims[0] : 1;
    const uint64_t sy = g.stride[nd - 2], sz = nd == 3 ? g.stride[0] : 0;
    const uint64_t nby = g.nblk[nd - 2], nbz = nd == 3 ? g.nblk[0] : 1;
    const uint64_t ntx = ceil_div(X, W), nyg = ceil_div(nby, nyb), ntask = ntx * nyg * nbz;
    const double two_eb = st->two_eb;
    const double rcp = __drcp_rn(two_eb);
    const int r = (int)(cap >> 1);
    const bool seg0 = ONE ? lane % bx == 0 : lane == 0;
    // int32 path: the field's described range bounds every |q| below 2^27
    // (abs-mode calls skip the describe: fp64 path)
    bool ip = false;
    if (KIND != 2 && st->vmin_bits <= st->vmax_bits && !(st->flags & F_NONFINITE)) {
        const double lo = KIND == 0 ? (double)ord2f((uint32_t)st->vmin_bits) : ord2d(st->vmin_bits);
        const double hi = KIND == 0 ? (double)ord2f((uint32_t)st->vmax_bits) : ord2d(st->vmax_bits);
        ip = fmax(fabs(lo), fabs(hi)) * rcp < 134217724.0;
    }
    bool bad = false;
    uint32_t cnt = 0;
    for (uint64_t t = blockIdx.x * (uint64_t)(blockDim.x >> 5) + warp; t < ntask;
         t += (uint64_t)gridDim.x * (blockDim.x >> 5)) {
        const uint64_t tx = t % ntx, t2 = t / ntx, cyg = t2 % nyg, cz = t2 / nyg;
        const uint64_t x0 = tx * W;
        const uint32_t lim = (uint32_t)umin(W, X - x0);
        const uint32_t nz = (uint32_t)umin(bz, Z - cz * bz);
        const uint64_t cy1 = umin(cyg * nyb + nyb, nby);
        for (uint64_t cy = cyg * nyb; cy < cy1; cy++) {
            const uint32_t ny = (uint32_t)umin(by, Y - cy * by);
            const uint32_t nit = nz * ny * steps;
            const uint64_t base = cz * bz * sz + cy * by * sy + x0;
            const uint64_t zjump = sz - (uint64_t)(ny - 1) * sy;
            uint64_t lrow = base, prow = base;
            uint32_t ls = 0, ly = 0, lit = 0, ps = 0, py = 0, pz = 0;
            double cd4[4] = {0.0, 0.0, 0.0, 0.0};   // previous segment's lane 31 (q, bb, cc, dd)
            int ci[4] = {0, 0, 0, 0};
            // cp.async ring: iteration lit's element lands in slot lit % kStripPf
            auto issue = [&]() {
                if (lit < nit) {
                    const uint32_t c = ONE ? lane : ls * 32 + lane;
                    const raw_t* src = (const raw_t*)in + lrow + (c < lim ? c : 0);
                    const uint32_t dst = ring_s + ((lit % kStripPf) * 32) * (uint32_t)sizeof(raw_t);
                    if (sizeof(raw_t) == 4)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src),
                                     "r"(c < lim ? 4 : 0) : "memory");
                    else
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
                                     "r"(c < lim ? 8 : 0) : "memory");
                    if (ONE || ++ls == steps) {
                        ls = 0;
                        if (++ly == ny) { ly = 0; lrow += zjump; } else lrow += sy;
                    }
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
                lit++;
            };
#pragma unroll 1
            for (int j = 0; j < kStripPf; j++) issue();
#pragma unroll 1
            for (uint32_t it = 0; it < nit; it++) {
                asm volatile("cp.async.wait_group %0;" ::"n"(kStripPf - 1) : "memory");
                const raw_t raw = ring[(it % kStripPf) * 32];
                {
                    const uint32_t s = ONE ? 0 : ps, y = py, z = pz;
                    const uint64_t rb = prow;
                    if (ONE || ++ps == steps) {
                        ps = 0;
                        if (++py == ny) { py = 0; pz++; prow += zjump; } else prow += sy;
                    }
                    const uint32_t c = s * 32 + lane;
                    const bool valid = c < lim;
                    const double q = valid ? q_of<KIND>(raw, two_eb, rcp, bad) : 0.0;
                    issue();   // iteration it + kStripPf into the slot just consumed
                    uint32_t code;
                    if (ip) {   // every |q| < 2^27: the fp64 sums below are exact, so int32 gives the same
                        const int qi = (int)q;
                        code = code_of_int(qi - strip_pred<int, ONE>(nd, qi, R, D, P, s, y, z, steps, seg0, lane,
                                                                     ci[0], ci[1], ci[2], ci[3]), r);
                    } else {
                        code = code_of_f64(__dsub_rn(q, strip_pred<double, ONE>(nd, q, R, D, P, s, y, z, steps, seg0,
                                                                                 lane, cd4[0], cd4[1], cd4[2], cd4[3])), r);
                    }
                    if (valid) {
                        codes[rb + c] = (uint16_t)code;
                        hist_add(h, code);
                    }
                    if (++cnt == 200) {   // 8-bit packed counters (warp-uniform count)
                        hist_flush(h);
                        cnt = 0;
                    }
                }
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
        }
    }
    hist_flush(h);
    if (bad) atomicOr(&st->flags, (unsigned long long)F_NONFINITE);
    hist_finish(h);
}

__global__ void prequantize_kernel(const void* __restrict__ in, int dtype, uint64_t n,
                                   const DevStatus* st, double* __restrict__ out) {
    const double two_eb = st->two_eb;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double v = dtype == 0 ? (double)((const float*)in)[i] : ((const double*)in)[i];
        out[i] = prequant(v, two_eb);
    }
}

template <int KIND>
int launch_kind(sdqz_ctx* ctx, const void* d_in, int ndims, const uint64_t dims[3],
                const uint32_t block[3], uint32_t cap, uint16_t* d_codes,
                unsigned long long* d_hist, double* d_heads) {
    size_t smem = (d_hist && cap <= kSmemHistMax) ? cap * sizeof(uint32_t) : 0;
    ensure_smem(ctx, (const void*)dq3d_kernel<KIND>, smem);
    ensure_smem(ctx, (const void*)dq2d_kernel<KIND>, smem);
    ensure_smem(ctx, (const void*)dq1d_kernel<KIND>, smem);
    ensure_smem(ctx, (const void*)dq_generic_kernel<KIND>, smem);
    uint64_t n = dims[0] * dims[1] * dims[2];
    int max_grid = ctx->num_sms * 8;
    // TMA-fed 3D path: fp32, 16-byte aligned base and row pitch, extents TMA can address
    if (KIND == 0 && ndims == 3 && is_fast_shape(ndims, block) && dims[2] % 4 == 0 &&
        ((uintptr_t)d_in & 15) == 0 && dims[2] < (1ull << 31) && dims[1] < (1ull << 31) &&
        dims[0] < (1ull << 31) && dims[1] * dims[2] < (1ull << 28) && !env_disabled("SDQZ_NO_TMA")) {
        CUtensorMap map;
        const uint64_t gd[3] = {dims[2], dims[1], dims[0]};
        const uint64_t gs[2] = {dims[2] * 4, dims[2] * dims[1] * 4};
        const uint32_t box[3] = {32, 8, 2};
        if (make_tensor_map(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d_in, gd, gs, box)) {
            const size_t tsm = kTmaWarps * kStages * kPair * 4 + kTmaWarps * kStages * 8 +
                               kTmaWarps * kHot * 32 * 4 + smem;
            ensure_smem(ctx, (const void*)dq3d_tma_kernel, tsm);
            const uint64_t ntask =
                ceil_div(ceil_div(dims[2], 8), 4) * ceil_div(dims[1], 8) * ceil_div(dims[0], 8);
            int per_sm = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dq3d_tma_kernel, kTmaWarps * 32, tsm);
            if (per_sm < 1) per_sm = 1;
            uint64_t grid = ceil_div(ntask, kTmaWarps);
            if (grid > (uint64_t)ctx->num_sms * per_sm) grid = (uint64_t)ctx->num_sms * per_sm;
            dq3d_tma_kernel<<<(unsigned)grid, kTmaWarps * 32, tsm, ctx->stream>>>(
                map, (const float*)d_in, dims[0], dims[1], dims[2], cap, ctx->d_status, d_codes, d_hist);
            SDQZ_LAUNCHED_NAMED(ctx, "dq3d_tma_kernel");
            return SDQZ_OK;
        }
    }
    // vectorised 1D path: whole 1024-point tasks, then the tail by dq1d_kernel
    if (dq1d_vec_span(KIND, ndims, dims, block, d_in, d_codes)) {
        const uint64_t nt = dims[0] / kVecTask;
        const size_t vsm = kWarpsPerCta * kHot * 32 * 4 + smem;
        ensure_smem(ctx, (const void*)dq1d_vec_kernel<true>, vsm);
        ensure_smem(ctx, (const void*)dq1d_vec_kernel<false>, vsm);
        uint64_t grid = ceil_div(nt, kWarpsPerCta);
        if (grid > (uint64_t)ctx->num_sms * 2) grid = (uint64_t)ctx->num_sms * 2;
        if (smem)
            dq1d_vec_kernel<true><<<(unsigned)grid, kThreads, vsm, ctx->stream>>>(
                (const float*)d_in, nt, cap, ctx->d_status, d_codes, d_hist, d_heads);
        else
            dq1d_vec_kernel<false><<<(unsigned)grid, kThreads, vsm, ctx->stream>>>(
                (const float*)d_in, nt, cap, ctx->d_status, d_codes, d_hist, d_heads);
        SDQZ_LAUNCHED_NAMED(ctx, "dq1d_vec_kernel");
        const uint64_t off = nt * kVecTask;
        if (off < dims[0]) {
            dq1d_kernel<0><<<1, kThreads, smem, ctx->stream>>>((const float*)d_in + off, dims[0] - off,
                                                               cap, ctx->d_status, d_codes + off, d_hist);
            SDQZ_LAUNCHED_NAMED(ctx, "dq1d_kernel");
        }
        return SDQZ_OK;
    }
    // vectorised 2D path (16-byte aligned rows)
    if (KIND == 0 && ndims == 2 && is_fast_shape(ndims, block) && dims[1] % 4 == 0 &&
        ((uintptr_t)d_in & 15) == 0 && ((uintptr_t)d_codes & 7) == 0 && !env_disabled("SDQZ_NO_VEC2D")) {
        const uint64_t nt = ceil_div(dims[1], 128) * ceil_div(dims[0], 16);
        const size_t vsm = kWarpsPerCta * kHot * 32 * 4 + smem;
        ensure_smem(ctx, (const void*)dq2d_vec_kernel<true>, vsm);
        ensure_smem(ctx, (const void*)dq2d_vec_kernel<false>, vsm);
        uint64_t grid = ceil_div(nt, kWarpsPerCta);
        if (grid > (uint64_t)ctx->num_sms * 2) grid = (uint64_t)ctx->num_sms * 2;
        if (smem)
            dq2d_vec_kernel<true><<<(unsigned)grid, kThreads, vsm, ctx->stream>>>(
                (const float*)d_in, dims[0], dims[1], cap, ctx->d_status, d_codes, d_hist);
        else
            dq2d_vec_kernel<false><<<(unsigned)grid, kThreads, vsm, ctx->stream>>>(
                (const float*)d_in, dims[0], dims[1], cap, ctx->d_status, d_codes, d_hist);
        SDQZ_LAUNCHED_NAMED(ctx, "dq2d_vec_kernel");
        return SDQZ_OK;
    }
    if (is_fast_shape(ndims, block)) {
        uint64_t ntask;
        if (ndims == 3) ntask = ceil_div(ceil_div(dims[2], 8), 4) * ceil_div(dims[1], 8) * ceil_div(dims[0], 8);
        else if (ndims == 2) ntask = ceil_div(ceil_div(dims[1], 16), 2) * ceil_div(dims[0], 16);
        else ntask = ceil_div(dims[0], 512);
        // persistent: 2 resident CTAs per SM (__launch_bounds__(256, 2)), each
        // walking many tasks, so the per-CTA histogram setup/merge amortizes
        uint64_t grid = ceil_div(ntask, kWarpsPerCta);
        if (grid > (uint64_t)ctx->num_sms * 2) grid = ctx->num_sms * 2;
        if (grid < 1) grid = 1;
        if (ndims == 3)
            dq3d_kernel<KIND><<<(unsigned)grid, kThreads, smem, ctx->stream>>>(
                d_in, dims[0], dims[1], dims[2], cap, ctx->d_status, d_codes, d_hist);
        else if (ndims == 2)
            dq2d_kernel<KIND><<<(unsigned)grid, kThreads, smem, ctx->stream>>>(
                d_in, dims[0], dims[1], cap, ctx->d_status, d_codes, d_hist);
        else
            dq1d_kernel<KIND><<<(unsigned)grid, kThreads, smem, ctx->stream>>>(
                d_in, dims[0], cap, ctx->d_status, d_codes, d_hist);
    } else {
        Geo g;
        g.nd = ndims;
        for (int a = 0; a < 3; a++) {
            g.dims[a] = a < ndims ? dims[a] : 1;
            g.block[a] = a < ndims ? block[a] : 1;
            g.nblk[a] = a < ndims ? ceil_div(dims[a], block[a]) : 1;
        }
        g.stride[ndims - 1] = 1;
        for (int a = ndims - 2; a >= 0; a--) g.stride[a] = g.stride[a + 1] * dims[a + 1];
        const uint32_t slots = blk_slots(ndims, block);
        const uint64_t nblocks_all = g.nblk[0] * g.nblk[1] * g.nblk[2];
        // few large blocks: thread per block-row segment (parallel, coalesced);
        // many small ones: thread per block (each point prequantized once)
        const char* rows_env = getenv("SDQZ_DQ_ROWS");
        const bool rows = rows_env ? rows_env[0] == '1'
                                   : (ndims == 1 ? block[0] >= 16 : nblocks_all < (uint64_t)ctx->num_sms * 2048);
        // 2D / 3D blocks of >= 128 points: warp per strip of block columns
        // (lane-private slots <= 12 KB a warp)
        uint64_t bpts = 1;
        for (int a = 0; a < ndims; a++) bpts *= block[a];
        const uint32_t bxx = block[ndims - 1];
        const uint32_t rw = bxx <= 32 ? (32 / bxx) * bxx : bxx, rsteps = (rw + 31) / 32;
        const uint64_t per_warp = (uint64_t)rsteps * (ndims == 3 ? 2 + block[ndims - 2] : 1);
        const char* strip_env = getenv("SDQZ_STRIP");
        const bool strip = ndims >= 2 && per_warp <= 48 && !env_disabled("SDQZ_NO_BLK") &&
                           (strip_env ? strip_env[0] == '1' : bpts >= 128);
        if (strip) {
            const uint64_t iters = (uint64_t)rsteps * block[ndims - 2] * (ndims == 3 ? block[0] : 1);
            const uint32_t nyb = iters >= 32 ? 1 : (uint32_t)ceil_div(32, iters);
            const uint64_t ntask = ceil_div(dims[ndims - 1], rw) * ceil_div(g.nblk[ndims - 2], nyb) *
                                   (ndims == 3 ? g.nblk[0] : 1);
            uint64_t grid = ceil_div(ntask, 8);
            if (grid > (uint64_t)ctx->num_sms * 8) grid = (uint64_t)ctx->num_sms * 8;
            if (grid < 1) grid = 1;
            const uint32_t hist_bytes = (uint32_t)((smem + 15) & ~(size_t)15);
            const size_t dsm = hist_bytes + (size_t)8 * per_warp * 32 * 8 + (size_t)8 * kStripPf * 32 * (KIND == 0 ? 4 : 8);
#define DQ_STRIP(ONE, ND)                                                                               \
            ensure_smem(ctx, (const void*)dq_strip_kernel<KIND, ONE, ND>, dsm);                         \
            dq_strip_kernel<KIND, ONE, ND><<<(unsigned)grid, 256, dsm, ctx->stream>>>(                  \
                d_in, g, rw, rsteps, nyb, cap, hist_bytes, ctx->d_status, d_codes, d_hist);
            if (ndims == 3) {
                if (rsteps == 1) { DQ_STRIP(true, 3) } else { DQ_STRIP(false, 3) }
            } else {
                if (rsteps == 1) { DQ_STRIP(true, 2) } else { DQ_STRIP(false, 2) }
            }
#undef DQ_STRIP
            SDQZ_LAUNCHED_NAMED(ctx, "dq_strip_kernel");
            return SDQZ_OK;
        }
        if (rows && !env_disabled("SDQZ_NO_BLK")) {
            const uint64_t nitems = ndims == 1 ? dims[0] : (n / dims[ndims - 1]) * g.nblk[ndims - 1];
            uint64_t grid = ceil_div(nitems, 256);
            if (grid > (uint64_t)ctx->num_sms * 16) grid = (uint64_t)ctx->num_sms * 16;
            if (grid < 1) grid = 1;
#define DQ_ROWS(ND)                                                                                     \
            ensure_smem(ctx, (const void*)dq_rows_kernel<KIND, ND>, smem);                              \
            dq_rows_kernel<KIND, ND><<<(unsigned)grid, 256, smem, ctx->stream>>>(d_in, g, nitems, cap,  \
                                                                                ctx->d_status, d_codes, d_hist);
            if (ndims == 3) { DQ_ROWS(3) } else if (ndims == 2) { DQ_ROWS(2) } else { DQ_ROWS(1) }
#undef DQ_ROWS
            SDQZ_LAUNCHED_NAMED(ctx, "dq_rows_kernel");
            return SDQZ_OK;
        }
        if (slots <= kBlkMaxSlots && !env_disabled("SDQZ_NO_BLK")) {
            // thread per block; 64 threads per CTA while the slots stay <= 1 KB per thread
            const uint32_t T = slots * 8 <= 1024 ? 64 : 32;
            const uint32_t hist_bytes = (uint32_t)((smem + 15) & ~(size_t)15);
            const size_t dsm = hist_bytes + (size_t)T * slots * 8;
            const uint64_t nblocks = g.nblk[0] * g.nblk[1] * g.nblk[2];
            uint64_t grid = ceil_div(nblocks, T);
            if (grid > (uint64_t)ctx->num_sms * 64) grid = (uint64_t)ctx->num_sms * 64;
            if (grid < 1) grid = 1;
#define DQ_BLOCKS(ND)                                                                                   \
            ensure_smem(ctx, (const void*)dq_blocks_kernel<KIND, ND>, dsm);                             \
            dq_blocks_kernel<KIND, ND><<<(unsigned)grid, T, dsm, ctx->stream>>>(d_in, g, cap, hist_bytes, \
                                                                              ctx->d_status, d_codes, d_hist);
            if (ndims == 3) { DQ_BLOCKS(3) } else if (ndims == 2) { DQ_BLOCKS(2) } else { DQ_BLOCKS(1) }
#undef DQ_BLOCKS
            SDQZ_LAUNCHED_NAMED(ctx, "dq_blocks_kernel");
            return SDQZ_OK;
        }
        uint64_t grid = ceil_div(n, kThreads);
        if (grid > (uint64_t)max_grid) grid = max_grid;
        if (grid < 1) grid = 1;
        dq_generic_kernel<KIND><<<(unsigned)grid, kThreads, smem, ctx->stream>>>(
            d_in, g, n, cap, ctx->d_status, d_codes, d_hist);
    }
    SDQZ_LAUNCHED_NAMED(ctx, !is_fast_shape(ndims, block) ? "dq_generic_kernel"
                             : ndims == 3 ? "dq3d_kernel" : ndims == 2 ? "dq2d_kernel" : "dq1d_kernel");
    return SDQZ_OK;
}

}  // namespace

bool env_disabled(const char* name) {
    const char* v = getenv(name);
    return v && v[0] && v[0] != '0';
}

bool make_tensor_map(CUtensorMap* map, CUtensorMapDataType dtype, uint32_t rank, const void* base,
                     const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box) {
    // resolved once per process (thread-safe static initialisation)
    static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return (PFN_cuTensorMapEncodeTiled_v12000)fn;
        cudaGetLastError();
        return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    }();
    if (!encode) return false;
    cuuint64_t gd[5], gs[4];
    cuuint32_t bx[5], es[5];
    for (uint32_t i = 0; i < rank; i++) {
        gd[i] = dims[i];
        bx[i] = box[i];
        es[i] = 1;
        if (i + 1 < rank) gs[i] = strides_bytes[i];
    }
    CUresult r = encode(map, dtype, rank, const_cast<void*>(base), gd, gs, bx, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool is_fast_shape(int ndims, const uint32_t block[3]) {
    if (ndims == 3) return block[0] == 8 && block[1] == 8 && block[2] == 8;
    if (ndims == 2) return block[0] == 16 && block[1] == 16;
    return ndims == 1 && block[0] == 32;
}

uint64_t dq1d_vec_span(int in_kind, int ndims, const uint64_t dims[3], const uint32_t block[3],
                       const void* d_in, const uint16_t* d_codes) {
    if (in_kind == 0 && ndims == 1 && is_fast_shape(ndims, block) && dims[0] >= kVecTask &&
        ((uintptr_t)d_in & 15) == 0 && ((uintptr_t)d_codes & 7) == 0 && !env_disabled("SDQZ_NO_VEC1D"))
        return dims[0] / kVecTask * kVecTask;
    return 0;
}

int launch_dualquant(sdqz_ctx* ctx, const void* d_in, int in_kind, int ndims,
                     const uint64_t dims[3], const uint32_t block[3], uint32_t cap,
                     uint16_t* d_codes, unsigned long long* d_hist, double* d_heads) {
    switch (in_kind) {
        case 0: return launch_kind<0>(ctx, d_in, ndims, dims, block, cap, d_codes, d_hist, d_heads);
        case 1: return launch_kind<1>(ctx, d_in, ndims, dims, block, cap, d_codes, d_hist, nullptr);
        default: return launch_kind<2>(ctx, d_in, ndims, dims, block, cap, d_codes, d_hist, nullptr);
    }
}

int launch_prequantize(sdqz_ctx* ctx, const void* d_in, int dtype, uint64_t n, double* d_out) {
    uint64_t grid = ceil_div(n, 256);
    if (grid > (uint64_t)ctx->num_sms * 8) grid = ctx->num_sms * 8;
    if (grid < 1) grid = 1;
    prequantize_kernel<<<(unsigned)grid, 256, 0, ctx->stream>>>(d_in, dtype, n, ctx->d_status, d_out);
    SDQZ_LAUNCHED_NAMED(ctx, "prequantize_kernel");
    return SDQZ_OK;
}

}  // namespace sdqz
