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

}  // namespace

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
