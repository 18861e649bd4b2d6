// common.cuh -- shared device helpers, the device status block and the context.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sdqz_cuda.h"

namespace sdqz {

constexpr int kWarp = 32;
constexpr uint32_t kFull = 0xffffffffu;
constexpr int kLutBits = 12;          // decode LUT width (entries = 4096)
constexpr int kMaxBw = 56;            // huffman.py:29 MAX_CODEWORD_BITS

// ---------------------------------------------------------------------------
// Device status block: every kernel reports errors/sizes here; the host reads
// it back once per call and raises the first error in the reference's order.
// ---------------------------------------------------------------------------
enum : uint32_t {
    F_NONFINITE = 1u << 0,      // resolve_error_bound: NaN/Inf      (core.py:163-164)
    F_RANGE_ZERO = 1u << 1,     // valrel on a constant field        (core.py:170-174)
    F_CODE_RANGE = 1u << 2,     // histogram/encode: code >= cap      (huffman.py:87-88)
    F_ABSENT_SYM = 1u << 3,     // encode: zero entry                 (huffman.py:201-202)
    F_ZERO_WIDTH = 1u << 4,     // deflate: packed unit bw 0          (huffman.py:235-236)
    F_ALL_ZERO_HIST = 1u << 5,  // build_tree: all-zero               (huffman.py:108-109)
    F_BW_TOO_BIG = 1u << 6,     // bitwidth > 56                      (huffman.py:138-142)
    F_KRAFT = 1u << 7,          // Kraft equality                     (huffman.py:161-164)
    F_NO_PRESENT = 1u << 8,     // empty bitwidth table               (huffman.py:154-155)
    F_OUT_RANGE = 1u << 9,      // outlier index >= n                 (archive.py:222-223)
    F_OUT_ORDER = 1u << 10,     // outlier indices not ascending      (archive.py:224-225)
    F_OUT_NONZERO = 1u << 11,   // codes[idx] != 0                    (dualquant.py:290-291)
    F_OUT_SLOW = 1u << 12,      // some outlier needs the fp64 path (not an error)
    F_OVERFLOW = 1u << 13,      // capacity exceeded (internal)
};

struct DevStatus {
    unsigned long long flags;
    unsigned long long decode_key;   // min over (step << 2 | kind), inflate errors
    unsigned long long n_zero;       // zero codes seen (inflate)
    unsigned long long vmin_bits;    // describe: ordered-int encoded min
    unsigned long long vmax_bits;    // describe: ordered-int encoded max
    unsigned long long payload_bytes;
    unsigned long long n_outliers;
    unsigned long long max_bw;
    unsigned long long n_present;
    unsigned long long bad_count;    // auxiliary value for messages
    unsigned long long bad_value;
    double eb;                       // resolved error bound (device-computed)
    double two_eb;
    unsigned long long pad[3];
};

// Decode kinds for decode_key (ordering matches the reference's lockstep checks).
enum : uint32_t { DK_NO_CODEWORD = 0, DK_EXHAUSTED = 1, DK_DISAGREE = 2 };

// Codebook tables produced on device (huffman.py:32-65).
struct BookDev {
    uint64_t* entries;     // [cap]  packed (bw << (unit-8)) | codeword
    uint8_t* bw;           // [cap]
    uint64_t* first;       // [58]
    int64_t* offsets;      // [59]
    uint32_t* symbols;     // [cap]
    uint32_t* lut;         // [1 << kLutBits] decode LUT
};

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

__host__ __device__ __forceinline__ uint64_t umin(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// ordered-int encodings so that atomicMin/Max on integers order floats
__device__ __forceinline__ uint32_t f2ord(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ inline float ord2f(uint32_t u) {
    uint32_t v = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    float f;
    memcpy(&f, &v, 4);
    return f;
}
__device__ __forceinline__ unsigned long long d2ord(double d) {
    unsigned long long u = (unsigned long long)__double_as_longlong(d);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ inline double ord2d(unsigned long long u) {
    unsigned long long v = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
    double d;
    memcpy(&d, &v, 8);
    return d;
}

// prequantize one value exactly as dualquant.py:76-77 (IEEE RN division,
// floor(|x| + 0.5), copysign).  Intrinsics keep the compiler from contracting.
__device__ __forceinline__ double prequant(double v, double two_eb) {
    double x = __ddiv_rn(v, two_eb);
    double r = floor(__dadd_rn(fabs(x), 0.5));
    return copysign(r, x);
}

// prequant() at a fraction of the FP64 cost, branch-free, for |v / 2eb| < 2^27
// (the caller checks that bound per warp).  y = v * RN(1/2eb) is within 2.5
// ulp of RN(v / 2eb); since |y| + 0.5 and its fraction are exact in fp64 here,
// floor(|y| + 0.5) can differ from the reference only when that fraction is
// within 2.5 ulp(2^27) < 2^-22 of 0 or 1.  Such a value ORs `amb`, and the
// caller then redoes the whole task with exact division.
__device__ __forceinline__ int prequant_int_fast(float v, double rcp, bool& amb) {
    const double y = __dmul_rn((double)v, rcp);
    const double t = __dadd_rn(fabs(y), 0.5);
    const double fl = floor(t);
    const double fr = __dsub_rn(t, fl);
    amb |= (fr < 2.384185791015625e-07) | (fr > 1.0 - 2.384185791015625e-07);
    const int m = (int)fl;
    return y < 0.0 ? -m : m;
}

// Warp-collective: the fast path, with the (rare) tie-neighbourhood lanes
// redone by exact division behind a warp-uniform branch.
__device__ __forceinline__ int prequant_int(float v, double rcp, double two_eb) {
    bool amb = false;
    int d = prequant_int_fast(v, rcp, amb);
    if (__any_sync(kFull, amb)) {
        if (amb) d = (int)prequant((double)v, two_eb);
    }
    return d;
}

__device__ __forceinline__ int warp_excl_scan(int v, int* total) {
    int lane = lane_id();
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    *total = __shfl_sync(kFull, x, 31);
    return x - v;
}

}  // namespace sdqz

// ---------------------------------------------------------------------------
// Context (opaque to callers).  Owns a stream, a grow-only scratch arena and
// the pinned status block.
// ---------------------------------------------------------------------------
// Reconstruction quality fused into the reconstruct kernels' epilogue
// (metrics.py:52-76; sdqz_decompress_quality): the original field, and one
// 5-double partial {sum d^2, max |d|, min orig, max orig, nonfinite} per CTA.
struct QualArgs {
    const void* orig = nullptr;   // nullptr: off
    int okind = 0;                // 0 f32, 1 f64
    double* part = nullptr;
    uint64_t nparts = 0;          // set by the launcher that fused it (0: not fused)
};

struct sdqz_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    uint64_t launches = 0;
    int num_sms = 148;

    sdqz::DevStatus* d_status = nullptr;   // device
    sdqz::DevStatus* h_status = nullptr;   // pinned host mirror
    void* h_stage = nullptr;               // pinned staging for host-buffer section copies
    size_t h_stage_bytes = 0;

    struct Buf {
        void* p = nullptr;
        size_t bytes = 0;
    };
    std::vector<Buf> bufs;

    // state of the last fused compress (sections live in scratch buffers)
    sdqz_header last_hdr{};
    bool have_archive = false;
    uint64_t archive_gen = 0;   // id of the last compress's archive (0: none);
                                // handles holding another id are stale

    // sharded compress in progress (sdqz_shard_quantize -> sdqz_shard_encode)
    struct Shard {
        const void* d_in = nullptr;
        int dtype = 0, eb_mode = 0, ndims = 0;
        double eb = 0;
        uint32_t cap = 0;
        uint64_t n = 0;
        uint64_t dims[3] = {1, 1, 1};
        uint32_t block[3] = {1, 1, 1};
        bool ready = false;
    } shard;

    // captured pipelines (CUDA graphs), valid while the scratch arena's
    // generation is unchanged
    struct Graph {
        cudaGraphExec_t exec = nullptr;
        std::string key;
        uint64_t gen = 0;
        uint64_t nlaunch = 0;
    };
    uint64_t gen = 0;
    Graph g_comp, g_decomp;
    std::string last_comp_key, last_decomp_key;
    uint64_t graph_replays = 0;
    cudaStream_t cap_stream = nullptr;   // capture stream
    cudaStream_t side = nullptr;         // forked branch (outlier lookup index beside the decode)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;

    // optional per-kernel device timer (bench / profiling)
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<const char*, size_t>> marks;   // (name, event index)
    std::vector<std::pair<std::string, double>> ktotals; // accumulated ms per kernel
    QualArgs qual;                                     // fused-quality request (sdqz_decompress_quality)
};

namespace sdqz {

// Named scratch slots (each grows on demand, never shrinks).
enum Slot : int {
    S_CODES = 0, S_HIST, S_BW, S_ENTRIES, S_FIRST, S_OFFSETS, S_SYMBOLS, S_LUT,
    S_CHUNK_BITS, S_CHUNK_AUX, S_BYTE_OFF, S_OUT_OFF, S_PAYLOAD, S_OUTREC, S_SORT,
    S_TREE, S_STAGE, S_DENSE, S_WORK, S_BLOCKFLAG, S_MISC, S_REDO, S_DTAB, S_COUNTER, S_QUAL, S_REBASE,
    S_HEADS,              // 1D block-head outlier values (dq1d_vec -> packer)
    S_HOST_A, S_HOST_B,   // device copies of host-buffer inputs / outputs (sdqz_*_host)
    S_NSLOTS
};

int set_error(sdqz_ctx* ctx, int code, const std::string& msg);
int cuda_check(sdqz_ctx* ctx, cudaError_t e, const char* what);
void* scratch(sdqz_ctx* ctx, int slot, size_t bytes, cudaError_t* e);
int fetch_status(sdqz_ctx* ctx);      // D2H of the status block + sync
int reset_status(sdqz_ctx* ctx);      // memset status on stream
int enqueue_status_copy(sdqz_ctx* ctx);   // D2H of the status block (no sync)
int sync_status(sdqz_ctx* ctx);           // stream sync (+ timer flush)
int reset_status_eb(sdqz_ctx* ctx, double eb, bool has_eb);   // ... and set eb / 2eb
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies per device: raise a
// kernel's limit on the context's device to >= bytes (remembered per
// (kernel, device) under a lock).
void ensure_smem(const sdqz_ctx* ctx, const void* func, size_t bytes);
uint64_t next_archive_gen();   // process-unique archive ids

#define SDQZ_CUDA(ctx, expr)                                                      \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess) return ::sdqz::cuda_check((ctx), _e, #expr);       \
    } while (0)

// After every kernel launch: count it, surface launch errors, and (when the
// context's kernel timer is on) record an event named after the kernel.  The
// time between consecutive marks on the context's single stream is that
// kernel's device time (host gaps are marked separately at syncs).
void kt_mark(sdqz_ctx* ctx, const char* name);

#define SDQZ_LAUNCHED_NAMED(ctx, name)                                            \
    do {                                                                          \
        (ctx)->launches++;                                                        \
        cudaError_t _e = cudaGetLastError();                                      \
        if (_e != cudaSuccess) return ::sdqz::cuda_check((ctx), _e, "kernel launch"); \
        if ((ctx)->timing) ::sdqz::kt_mark((ctx), (name));                        \
    } while (0)

template <typename T>
T* scratch_as(sdqz_ctx* ctx, int slot, size_t count, int* rc) {
    cudaError_t e = cudaSuccess;
    void* p = scratch(ctx, slot, count * sizeof(T), &e);
    if (!p) *rc = cuda_check(ctx, e, "scratch allocation");
    return (T*)p;
}

}  // namespace sdqz
