// describe.cu -- K1: min / max / nonfinite scan of the input field
// (core.py:136-158) and device-side error-bound resolution (core.py:161-175).
//
// HBM-bound streaming reduction: 4N (f32) bytes read once with 16-byte
// vector loads, grid = 4 x SMs persistent CTAs, warp shuffles then one
// ordered-integer atomicMin/Max per CTA.
#include "kernels.cuh"

namespace sdqz {

namespace {

template <typename T>
struct VecOf;
template <>
struct VecOf<float> { using V = float4; static constexpr int W = 4; };
template <>
struct VecOf<double> { using V = double2; static constexpr int W = 2; };

__device__ __forceinline__ void acc(float v, float& mn, float& mx, bool& bad) {
    bad |= !isfinite(v);
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
}
__device__ __forceinline__ void acc(double v, double& mn, double& mx, bool& bad) {
    bad |= !isfinite(v);
    mn = fmin(mn, v);
    mx = fmax(mx, v);
}

template <typename T>
__global__ void __launch_bounds__(256) describe_kernel(const T* __restrict__ in, uint64_t n,
                                                       DevStatus* st) {
    using V = typename VecOf<T>::V;
    constexpr int W = VecOf<T>::W;
    T mn = (T)INFINITY, mx = (T)-INFINITY;
    bool bad = false;
    uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    // aligned prefix handled scalar
    uint64_t mis = ((uintptr_t)in / sizeof(T)) % W;
    uint64_t head = mis ? (W - mis) : 0;
    if (head > n) head = n;
    for (uint64_t i = tid; i < head; i += stride) acc(in[i], mn, mx, bad);
    const V* vin = reinterpret_cast<const V*>(in + head);
    uint64_t nv = (n - head) / W;
    auto accv = [&](const V& v) {
        if constexpr (W == 4) {
            acc(v.x, mn, mx, bad); acc(v.y, mn, mx, bad);
            acc(v.z, mn, mx, bad); acc(v.w, mn, mx, bad);
        } else {
            acc(v.x, mn, mx, bad); acc(v.y, mn, mx, bad);
        }
    };
    // full batches of kBatch unconditional loads in flight per thread
    constexpr int kBatch = 8;
    uint64_t i = tid;
    for (; i + (kBatch - 1) * stride < nv; i += kBatch * stride) {
        V v[kBatch];
#pragma unroll
        for (int k = 0; k < kBatch; k++) v[k] = __ldg(vin + i + k * stride);
#pragma unroll
        for (int k = 0; k < kBatch; k++) accv(v[k]);
    }
    for (; i < nv; i += stride) accv(__ldg(vin + i));
    for (uint64_t i = head + nv * W + tid; i < n; i += stride) acc(in[i], mn, mx, bad);

#pragma unroll
    for (int o = 16; o; o >>= 1) {
        T a = __shfl_xor_sync(kFull, mn, o), b = __shfl_xor_sync(kFull, mx, o);
        if constexpr (W == 4) { mn = fminf(mn, a); mx = fmaxf(mx, b); }
        else { mn = fmin(mn, a); mx = fmax(mx, b); }
    }
    bad = __any_sync(kFull, bad);
    __shared__ T smn[8], smx[8];
    __shared__ int sbad;
    if (threadIdx.x == 0) sbad = 0;
    __syncthreads();
    int w = threadIdx.x >> 5;
    if (lane_id() == 0) {
        smn[w] = mn;
        smx[w] = mx;
        if (bad) sbad = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); i++) {
            if constexpr (W == 4) { mn = fminf(mn, smn[i]); mx = fmaxf(mx, smx[i]); }
            else { mn = fmin(mn, smn[i]); mx = fmax(mx, smx[i]); }
        }
        // all-NaN blocks leave mn = +inf / mx = -inf: harmless, NaN => error anyway
        if constexpr (W == 4) {
            atomicMin(&st->vmin_bits, (unsigned long long)f2ord(mn));
            atomicMax(&st->vmax_bits, (unsigned long long)f2ord(mx));
        } else {
            atomicMin(&st->vmin_bits, d2ord(mn));
            atomicMax(&st->vmax_bits, d2ord(mx));
        }
        if (sbad) atomicOr(&st->flags, (unsigned long long)F_NONFINITE);
    }
}

// core.py:161-175 on device: eb = magnitude (abs) or magnitude * (max - min).
__global__ void resolve_kernel(DevStatus* st, int dtype, int eb_mode, double magnitude) {
    double vmin, vmax;
    if (dtype == 0) {
        vmin = (double)ord2f((uint32_t)st->vmin_bits);
        vmax = (double)ord2f((uint32_t)st->vmax_bits);
    } else {
        vmin = ord2d(st->vmin_bits);
        vmax = ord2d(st->vmax_bits);
    }
    double eb = magnitude;
    if (eb_mode == 1) {
        double rng = __dsub_rn(vmax, vmin);
        if (rng == 0.0) atomicOr(&st->flags, (unsigned long long)F_RANGE_ZERO);
        eb = __dmul_rn(magnitude, rng);
    }
    st->eb = eb;
    st->two_eb = __dmul_rn(2.0, eb);
}

// quality (metrics.py:52-76): one pass over (orig, recon) in fp64 -> per-CTA
// partials {sum d^2, max |d|, min a, max a, nonfinite(a)}; a single CTA then
// folds the partials in a fixed order (deterministic result).
constexpr int kQualCtas = 592;
template <typename A, typename B>
__global__ void __launch_bounds__(256) quality_partial_kernel(const A* __restrict__ a, const B* __restrict__ b,
                                                              uint64_t n, double* __restrict__ part) {
    double ss = 0.0, mx = 0.0, amin = INFINITY, amax = -INFINITY;
    bool bad = false;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double x = (double)__ldcs(a + i), y = (double)__ldcs(b + i);
        const double d = __dsub_rn(x, y);
        ss = __fma_rn(d, d, ss);
        mx = fmax(mx, fabs(d));
        amin = fmin(amin, x);
        amax = fmax(amax, x);
        bad |= !isfinite(x);
        mx = isnan(d) ? d : mx;   // a NaN difference propagates (numpy max)
    }
    __shared__ double s[5][8];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        ss += __shfl_down_sync(kFull, ss, o);
        const double m2 = __shfl_down_sync(kFull, mx, o);
        mx = isnan(m2) ? m2 : fmax(mx, m2);
        amin = fmin(amin, __shfl_down_sync(kFull, amin, o));
        amax = fmax(amax, __shfl_down_sync(kFull, amax, o));
    }
    const bool wbad = __any_sync(kFull, bad);
    if (lane == 0) { s[0][w] = ss; s[1][w] = mx; s[2][w] = amin; s[3][w] = amax; s[4][w] = wbad ? 1.0 : 0.0; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double r0 = 0.0, r1 = 0.0, r2 = INFINITY, r3 = -INFINITY, r4 = 0.0;
        for (int k = 0; k < 8; k++) {
            r0 += s[0][k];
            r1 = isnan(s[1][k]) ? s[1][k] : fmax(r1, s[1][k]);
            r2 = fmin(r2, s[2][k]);
            r3 = fmax(r3, s[3][k]);
            r4 = fmax(r4, s[4][k]);
        }
        double* p = part + 5 * blockIdx.x;
        p[0] = r0; p[1] = r1; p[2] = r2; p[3] = r3; p[4] = r4;
    }
}

__global__ void quality_final_kernel(const double* __restrict__ part, int nparts, double* __restrict__ out) {
    double r0 = 0.0, r1 = 0.0, r2 = INFINITY, r3 = -INFINITY, r4 = 0.0;
    for (int k = 0; k < nparts; k++) {
        const double* p = part + 5 * k;
        r0 += p[0];
        r1 = isnan(p[1]) ? p[1] : fmax(r1, p[1]);
        r2 = fmin(r2, p[2]);
        r3 = fmax(r3, p[3]);
        r4 = fmax(r4, p[4]);
    }
    out[0] = r0; out[1] = r1; out[2] = r2; out[3] = r3; out[4] = r4;
}

}  // namespace

int launch_quality_fold(sdqz_ctx* ctx, const double* d_part, uint64_t nparts, double* d_out) {
    quality_final_kernel<<<1, 1, 0, ctx->stream>>>(d_part, (int)nparts, d_out);
    SDQZ_LAUNCHED_NAMED(ctx, "quality_final_kernel");
    return SDQZ_OK;
}

int launch_quality(sdqz_ctx* ctx, const void* a, int a_dtype, const void* b, int b_dtype, uint64_t n,
                   double* d_part, double* d_out) {
    uint64_t g = ceil_div(n, 256 * 4);
    const int grid = (int)(g < 1 ? 1 : (g > (uint64_t)kQualCtas ? kQualCtas : g));
#define QK(TA, TB) quality_partial_kernel<TA, TB><<<grid, 256, 0, ctx->stream>>>((const TA*)a, (const TB*)b, n, d_part)
    if (a_dtype == 0 && b_dtype == 0) QK(float, float);
    else if (a_dtype == 0) QK(float, double);
    else if (b_dtype == 0) QK(double, float);
    else QK(double, double);
#undef QK
    SDQZ_LAUNCHED_NAMED(ctx, "quality_partial_kernel");
    quality_final_kernel<<<1, 1, 0, ctx->stream>>>(d_part, grid, d_out);
    SDQZ_LAUNCHED_NAMED(ctx, "quality_final_kernel");
    return SDQZ_OK;
}

int launch_describe(sdqz_ctx* ctx, const void* d_in, int dtype, uint64_t n) {
    int grid = ctx->num_sms * 4;
    uint64_t need = ceil_div(n, 256 * 8);
    if (need < (uint64_t)grid) grid = (int)(need ? need : 1);
    if (dtype == 0)
        describe_kernel<float><<<grid, 256, 0, ctx->stream>>>((const float*)d_in, n, ctx->d_status);
    else
        describe_kernel<double><<<grid, 256, 0, ctx->stream>>>((const double*)d_in, n, ctx->d_status);
    SDQZ_LAUNCHED_NAMED(ctx, "describe_kernel");
    return SDQZ_OK;
}

int launch_resolve(sdqz_ctx* ctx, int dtype, int eb_mode, double magnitude) {
    resolve_kernel<<<1, 1, 0, ctx->stream>>>(ctx->d_status, dtype, eb_mode, magnitude);
    SDQZ_LAUNCHED_NAMED(ctx, "resolve_kernel");
    return SDQZ_OK;
}

}  // namespace sdqz
