// scan.cuh -- one-CTA (1024 threads) exclusive scan of chunk byte lengths
// (ceil(bits / 8), huffman.py:245-246) and outlier counts into 64-bit chunk
// offsets; rows of 1024 chunks with coalesced loads/stores, the next row's
// loads issued before the current row's scan.  Totals go to the status block.
#pragma once
#include "common.cuh"

namespace sdqz {

__device__ __forceinline__ void block_chunk_scan(const uint32_t* __restrict__ chunk_bits,
                                                 const uint32_t* __restrict__ chunk_zeros, uint64_t C,
                                                 unsigned long long* __restrict__ byte_off,
                                                 unsigned long long* __restrict__ out_off,
                                                 unsigned long long payload_cap, bool records,
                                                 unsigned long long out_cap, DevStatus* st) {
    __shared__ unsigned long long wsb[32], wso[32];
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned long long carry_b = 0, carry_o = 0;
    uint32_t nb = tid < C ? chunk_bits[tid] : 0;
    uint32_t nz = (tid < C && chunk_zeros) ? chunk_zeros[tid] : 0;
    for (uint64_t r0 = 0; r0 < C; r0 += 1024) {
        const uint64_t i = r0 + tid;
        const uint32_t vb = (nb + 7) >> 3, vz = nz;
        const uint64_t ni = i + 1024;
        nb = ni < C ? chunk_bits[ni] : 0;
        nz = (ni < C && chunk_zeros) ? chunk_zeros[ni] : 0;
        unsigned long long xb = vb, xo = vz;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long yb = __shfl_up_sync(kFull, xb, o), yo = __shfl_up_sync(kFull, xo, o);
            if (lane >= (uint32_t)o) { xb += yb; xo += yo; }
        }
        if (lane == 31) { wsb[wid] = xb; wso[wid] = xo; }
        __syncthreads();
        if (wid == 0) {
            unsigned long long ub = wsb[lane], uo = wso[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long yb = __shfl_up_sync(kFull, ub, o), yo = __shfl_up_sync(kFull, uo, o);
                if (lane >= (uint32_t)o) { ub += yb; uo += yo; }
            }
            wsb[lane] = ub;
            wso[lane] = uo;
        }
        __syncthreads();
        if (i < C) {
            byte_off[i] = carry_b + (wid ? wsb[wid - 1] : 0) + xb - vb;
            if (out_off) out_off[i] = carry_o + (wid ? wso[wid - 1] : 0) + xo - vz;
        }
        carry_b += wsb[31];
        carry_o += wso[31];
        __syncthreads();
    }
    if (tid == 0) {
        st->payload_bytes = carry_b;
        st->n_outliers = carry_o;
        if (carry_b > payload_cap || (records && carry_o > out_cap))
            atomicOr(&st->flags, (unsigned long long)F_OVERFLOW);
    }
}

}  // namespace sdqz
