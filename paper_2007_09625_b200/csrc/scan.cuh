// scan.cuh -- one-CTA (1024 threads) exclusive scan of chunk byte lengths
// (ceil(bits / 8), huffman.py:245-246) and outlier counts into 64-bit chunk
// offsets; rows of 1024 chunks with coalesced loads/stores, the next row's
// loads issued before the current row's scan.  Totals go to the status block.
#pragma once
#include "common.cuh"
#include "tma.cuh"

namespace sdqz {

__device__ __forceinline__ void block_chunk_scan(const uint32_t* __restrict__ chunk_bits,
                                                 const uint32_t* __restrict__ chunk_zeros, uint64_t C,
                                                 unsigned long long* __restrict__ byte_off,
                                                 unsigned long long* __restrict__ out_off,
                                                 unsigned long long payload_cap, bool records,
                                                 unsigned long long out_cap, DevStatus* st) {
    // rows of 4096 chunks, 4 consecutive per thread (one 16-byte load, two
    // 16-byte stores per array: a warp's accesses are contiguous)
    __shared__ unsigned long long wsb[32], wso[32];
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const bool vec = (((uintptr_t)chunk_bits | (uintptr_t)chunk_zeros | (uintptr_t)byte_off |
                       (uintptr_t)out_off) & 15) == 0;
    unsigned long long carry_b = 0, carry_o = 0;
    // row r+1's loads are issued before row r is scanned
    auto load = [&](uint64_t i0, uint32_t (&vb)[4], uint32_t (&vz)[4]) {
        if (vec && i0 + 4 <= C) {
            const uint4 u = *reinterpret_cast<const uint4*>(chunk_bits + i0);
            vb[0] = u.x; vb[1] = u.y; vb[2] = u.z; vb[3] = u.w;
            if (chunk_zeros) {
                const uint4 z = *reinterpret_cast<const uint4*>(chunk_zeros + i0);
                vz[0] = z.x; vz[1] = z.y; vz[2] = z.z; vz[3] = z.w;
            } else {
                vz[0] = vz[1] = vz[2] = vz[3] = 0;
            }
        } else {
#pragma unroll
            for (int q = 0; q < 4; q++) {
                vb[q] = i0 + q < C ? chunk_bits[i0 + q] : 0;
                vz[q] = (i0 + q < C && chunk_zeros) ? chunk_zeros[i0 + q] : 0;
            }
        }
    };
    uint32_t nb[4], nz[4];
    load(4 * (uint64_t)tid, nb, nz);
    for (uint64_t r0 = 0; r0 < C; r0 += 4096) {
        const uint64_t i0 = r0 + 4 * (uint64_t)tid;
        uint32_t vb[4], vz[4];
#pragma unroll
        for (int q = 0; q < 4; q++) { vb[q] = nb[q]; vz[q] = nz[q]; }
        if (r0 + 4096 < C) load(i0 + 4096, nb, nz);
        unsigned long long tb = 0, to = 0;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            vb[q] = (vb[q] + 7) >> 3;
            tb += vb[q];
            to += vz[q];
        }
        unsigned long long xb = tb, xo = to;
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
        unsigned long long rb[4], ro[4];
        rb[0] = carry_b + (wid ? wsb[wid - 1] : 0) + xb - tb;
        ro[0] = carry_o + (wid ? wso[wid - 1] : 0) + xo - to;
#pragma unroll
        for (int q = 1; q < 4; q++) {
            rb[q] = rb[q - 1] + vb[q - 1];
            ro[q] = ro[q - 1] + vz[q - 1];
        }
        if (vec && i0 + 4 <= C) {
            reinterpret_cast<ulonglong2*>(byte_off + i0)[0] = make_ulonglong2(rb[0], rb[1]);
            reinterpret_cast<ulonglong2*>(byte_off + i0)[1] = make_ulonglong2(rb[2], rb[3]);
            if (out_off) {
                reinterpret_cast<ulonglong2*>(out_off + i0)[0] = make_ulonglong2(ro[0], ro[1]);
                reinterpret_cast<ulonglong2*>(out_off + i0)[1] = make_ulonglong2(ro[2], ro[3]);
            }
        } else {
#pragma unroll
            for (int q = 0; q < 4; q++) {
                if (i0 + q < C) {
                    byte_off[i0 + q] = rb[q];
                    if (out_off) out_off[i0 + q] = ro[q];
                }
            }
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


// ---------------------------------------------------------------------------
// Cluster version: the scan of one CTA is bound by that SM's store bandwidth
// (two u64 arrays, ~32 B/clk), so the chunks are spread over a cluster of
// kScanCtas CTAs (2048 chunks each per pass, 2 per thread).  Each pass: block
// scan, CTA totals exchanged through distributed shared memory (one cluster
// barrier; the total slots are double-buffered by pass parity), stores.
// ---------------------------------------------------------------------------
constexpr uint32_t kScanCtas = 8;
constexpr uint32_t kScanPer = 2048;   // chunks per CTA per pass

__device__ __forceinline__ void cluster_chunk_scan(uint32_t rank, const uint32_t* __restrict__ chunk_bits,
                                                   const uint32_t* __restrict__ chunk_zeros, uint64_t C,
                                                   unsigned long long* __restrict__ byte_off,
                                                   unsigned long long* __restrict__ out_off,
                                                   unsigned long long payload_cap, bool records,
                                                   unsigned long long out_cap, DevStatus* st) {
    __shared__ unsigned long long wsb[32], wso[32];
    __shared__ unsigned long long tot[2][2];        // [pass parity][bytes, outliers]
    __shared__ unsigned long long pre[2], ptot[2];  // this CTA's exclusive base, pass total
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const bool vec = (((uintptr_t)chunk_bits | (uintptr_t)chunk_zeros) & 7) == 0 &&
                     (((uintptr_t)byte_off | (uintptr_t)out_off) & 15) == 0;
    unsigned long long carry_b = 0, carry_o = 0;
    uint32_t par = 0;
    for (uint64_t base = 0; base < C; base += (uint64_t)kScanCtas * kScanPer, par ^= 1) {
        const uint64_t i0 = base + (uint64_t)rank * kScanPer + 2 * (uint64_t)tid;
        uint32_t vb[2], vz[2];
        if (vec && i0 + 2 <= C) {
            const uint2 u = *reinterpret_cast<const uint2*>(chunk_bits + i0);
            vb[0] = u.x; vb[1] = u.y;
            if (chunk_zeros) {
                const uint2 z = *reinterpret_cast<const uint2*>(chunk_zeros + i0);
                vz[0] = z.x; vz[1] = z.y;
            } else {
                vz[0] = vz[1] = 0;
            }
        } else {
#pragma unroll
            for (int q = 0; q < 2; q++) {
                vb[q] = i0 + q < C ? chunk_bits[i0 + q] : 0;
                vz[q] = (i0 + q < C && chunk_zeros) ? chunk_zeros[i0 + q] : 0;
            }
        }
        vb[0] = (vb[0] + 7) >> 3;
        vb[1] = (vb[1] + 7) >> 3;
        const unsigned long long tb = (unsigned long long)vb[0] + vb[1];
        const unsigned long long to = (unsigned long long)vz[0] + vz[1];
        unsigned long long xb = tb, xo = to;
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
            if (lane == 31) { tot[par][0] = ub; tot[par][1] = uo; }
        }
        // publish this CTA's totals to the cluster
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (wid == 0) {
            unsigned long long rb = 0, ro = 0;
            if (lane < kScanCtas) {
                const uint32_t local = smem_u32(&tot[par][0]);
                uint32_t remote;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(lane));
                asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(rb) : "r"(remote));
                asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(ro) : "r"(remote + 8));
            }
            unsigned long long sb = rb, so = ro;   // inclusive scan over ranks
#pragma unroll
            for (int o = 1; o < (int)kScanCtas; o <<= 1) {
                const unsigned long long yb = __shfl_up_sync(kFull, sb, o), yo = __shfl_up_sync(kFull, so, o);
                if (lane >= (uint32_t)o) { sb += yb; so += yo; }
            }
            const unsigned long long eb = __shfl_sync(kFull, sb - rb, rank), eo = __shfl_sync(kFull, so - ro, rank);
            const unsigned long long ab = __shfl_sync(kFull, sb, kScanCtas - 1),
                                     ao = __shfl_sync(kFull, so, kScanCtas - 1);
            if (lane == 0) { pre[0] = eb; pre[1] = eo; ptot[0] = ab; ptot[1] = ao; }
        }
        __syncthreads();
        unsigned long long r0b = carry_b + pre[0] + (wid ? wsb[wid - 1] : 0) + xb - tb;
        unsigned long long r0o = carry_o + pre[1] + (wid ? wso[wid - 1] : 0) + xo - to;
        if (vec && i0 + 2 <= C) {
            *reinterpret_cast<ulonglong2*>(byte_off + i0) = make_ulonglong2(r0b, r0b + vb[0]);
            if (out_off) *reinterpret_cast<ulonglong2*>(out_off + i0) = make_ulonglong2(r0o, r0o + vz[0]);
        } else {
#pragma unroll
            for (int q = 0; q < 2; q++) {
                if (i0 + q < C) {
                    byte_off[i0 + q] = r0b;
                    if (out_off) out_off[i0 + q] = r0o;
                }
                r0b += vb[q];
                r0o += vz[q];
            }
        }
        carry_b += ptot[0];
        carry_o += ptot[1];
        __syncthreads();   // wsb / pre reused by the next pass
    }
    if (rank == 0 && tid == 0) {
        st->payload_bytes = carry_b;
        st->n_outliers = carry_o;
        if (carry_b > payload_cap || (records && carry_o > out_cap))
            atomicOr(&st->flags, (unsigned long long)F_OVERFLOW);
    }
    // no CTA leaves while another may still read its totals
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

}  // namespace sdqz
