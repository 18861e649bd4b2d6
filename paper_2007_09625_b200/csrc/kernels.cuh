// kernels.cuh -- host-side launchers shared between translation units.
#pragma once
#include "common.cuh"

namespace sdqz {

// describe.cu ---------------------------------------------------------------
// min/max (ordered bits) and nonfinite flag into the status block.
int launch_describe(sdqz_ctx* ctx, const void* d_in, int dtype, uint64_t n);
// eb = magnitude (abs) or magnitude*(max-min) (valrel), computed on device
// from the describe results; sets F_RANGE_ZERO / F_NONFINITE accordingly.
int launch_resolve(sdqz_ctx* ctx, int dtype, int eb_mode, double magnitude);

// dualquant.cu --------------------------------------------------------------
// in_kind: 0 f32 data, 1 f64 data, 2 f64 prequantized units.  Reads two_eb from
// the status block.  d_hist (uint64[cap]) must be zeroed by the caller.
int launch_dualquant(sdqz_ctx* ctx, const void* d_in, int in_kind, int ndims,
                     const uint64_t dims[3], const uint32_t block[3], uint32_t cap,
                     uint16_t* d_codes, unsigned long long* d_hist, double* d_heads = nullptr);
// points [0, span) take the vectorised 1D dual-quant (block 32, 1024-point
// tasks) for this input: with d_heads it also stores the prequantized value of
// every block head whose code is an outlier at d_heads[i / 32], so the packer
// need not re-read the input there.  0 when that path does not apply.
uint64_t dq1d_vec_span(int in_kind, int ndims, const uint64_t dims[3], const uint32_t block[3],
                       const void* d_in, const uint16_t* d_codes);
int launch_prequantize(sdqz_ctx* ctx, const void* d_in, int dtype, uint64_t n, double* d_out);

// huffman.cu ----------------------------------------------------------------
int launch_histogram_u32(sdqz_ctx* ctx, const uint32_t* codes, uint64_t n, uint32_t cap,
                         unsigned long long* hist);
// tree + canonical book from a histogram (uint64[cap]).  bw_only: stop after
// the bitwidths (build_tree API).  from_bw: skip the tree, canonize d_bw.
// err_format: report table errors as archive-format errors (deserialize).
int launch_codebook(sdqz_ctx* ctx, const unsigned long long* d_hist, uint8_t* d_bw, uint32_t cap,
                    const BookDev& book, bool build_tree, bool canon, bool err_format);
// decode LUT from reverse tables (first/offsets/symbols, max_bw from status or arg)
int launch_build_lut(sdqz_ctx* ctx, const uint64_t* first, const int64_t* offsets,
                     const uint32_t* symbols, int max_bw_or_neg, uint32_t* lut);

// chunked encode/deflate from uint16 codes + packed entries (unit from status).
// Also compacts outliers (code 0) as interleaved {u64 idx, f64 value} records,
// recomputing the value from the input (in_kind as in launch_dualquant);
// d_in may be null when no outlier output is wanted.
struct DeflateJob {
    const uint16_t* codes = nullptr;     // source codes (uint16) ...
    const void* units = nullptr;         // ... or packed units (stage API deflate)
    int units_width = 0;                 // 32/64 when `units` is used
    uint64_t n = 0;
    uint32_t chunk = 0;
    const uint64_t* entries = nullptr;   // codebook (when codes are used)
    uint32_t cap = 0;
    uint32_t* chunk_bits = nullptr;      // [C]
    uint8_t* payload = nullptr;          // capacity payload_cap
    uint64_t payload_cap = 0;
    // outliers
    const void* in = nullptr;
    int in_kind = 0;
    uint64_t in_split = ~0ull;           // indices >= in_split read from `in_tail`
    const void* in_tail = nullptr;
    uint64_t idx_base = 0;               // added to every emitted index
    uint64_t rec_limit = ~0ull;          // records only for (job-local) indices below this
    void* out_records = nullptr;         // {u64, f64}[max]
    const double* heads = nullptr;       // outlier values of 1D block heads below heads_limit (dq1d_vec)
    uint64_t heads_limit = 0;
    uint64_t out_cap = 0;
    bool want_payload = true;
    bool trusted = false;                // codes came from K2 (< cap, all present in the book)
};
int launch_deflate(sdqz_ctx* ctx, const DeflateJob& job);

int launch_encode_u32(sdqz_ctx* ctx, const uint32_t* codes, uint64_t n, const uint64_t* entries,
                      uint32_t cap, int unit, void* units);

// inflate into uint16 (or uint32 when out32) codes; counts zero codes.
int launch_inflate(sdqz_ctx* ctx, const uint8_t* payload, uint64_t payload_bytes,
                   const uint32_t* chunk_bits, uint64_t n_chunks, uint32_t chunk,
                   const uint64_t* first, const int64_t* offsets, const uint32_t* symbols,
                   const uint32_t* lut, int max_bw, uint32_t cap, uint64_t n, void* codes, bool out32,
                   uint64_t stream_bytes = 0);   // the payload's own size when payload_bytes is a buffer capacity

// inflate.cu: decode tables (primary 12-bit + second level) and the warp-per-chunk
// self-synchronising decoder; chunks it cannot finish are flagged in `redo`.
// (old_lut, if non-null, also receives the sequential decoder's 12-bit table)
int launch_decode_prep(sdqz_ctx* ctx, const uint64_t* first, const int64_t* offsets,
                       const uint32_t* symbols, int max_bw, uint32_t** tab_out, uint32_t* old_lut,
                       const uint32_t* chunk_bits, uint64_t n_chunks, unsigned long long* byte_off,
                       uint8_t* redo, int ns);
// symbols per decode-table step (3 or 6) for a stream of n codes in payload_bytes
int decode_ns(uint64_t payload_bytes, uint64_t n);
int launch_inflate_fast(sdqz_ctx* ctx, const uint8_t* payload, uint64_t nwords,
                        const uint32_t* chunk_bits, const unsigned long long* byte_off,
                        uint64_t n_chunks, uint32_t chunk, uint64_t n, const uint64_t* first,
                        const int64_t* offsets, const uint32_t* symbols, const uint32_t* tab,
                        int max_bw, uint16_t* codes, uint8_t* redo, int ns);

// reconstruct.cu ------------------------------------------------------------
// Validate outlier records (range, order, code==0) and scatter their fp64
// bits into `dense` (uint64[n]); flag blocks needing the fp64 path.
// Outlier records by flat index for the reconstruct kernels (no dense side
// array): the records are sorted ascending (validated), bucketed by 1024
// points; a zero code at i binary-searches its bucket's records.
struct OutLookup {
    const unsigned long long* idx;     // record j's index at idx[j * stride]
    const unsigned long long* val;     // its f64 bits at val[j * stride]
    uint32_t stride;                   // 2: interleaved archive records, 1: separate arrays
    const unsigned long long* start;   // [ceil(n / 1024) + 1]: first record of each bucket
    uint64_t k;
    uint64_t base;                     // added to a query index (a kernel run on a sub-range)
    const unsigned long long* big;     // [1]: nonzero when some record's |value| >= 2^29 (or NaN)
};
// builds the bucket table (context scratch) for k records over n points
int launch_outlier_index(sdqz_ctx* ctx, const void* records, const uint64_t* idx, const double* val,
                         uint64_t k, uint64_t n, OutLookup* out);
// record checks (range, order, codes[idx] == 0) and fp64-path block flags
int launch_outlier_scatter(sdqz_ctx* ctx, const void* records, const uint64_t* idx,
                           const double* val, uint64_t k, uint64_t n, const uint16_t* codes,
                           int ndims, const uint64_t dims[3], const uint32_t block[3],
                           uint8_t* blockflag, bool check_format);
bool rq1d_records_ok(int ndims, const uint64_t dims[3], const uint32_t block[3], const void* codes,
                     const void* out, const void* records);
int launch_reconstruct_1d_records(sdqz_ctx* ctx, const uint16_t* codes, const void* records, uint64_t k,
                                  uint64_t n, uint32_t cap, double two_eb, void* out, int out_kind,
                                  uint8_t* blockflag);
// fixed-order fold of per-CTA quality partials (5 doubles each) into d_out[5]
int launch_quality_fold(sdqz_ctx* ctx, const double* d_part, uint64_t nparts, double* d_out);
int launch_quality(sdqz_ctx* ctx, const void* a, int a_dtype, const void* b, int b_dtype, uint64_t n,
                   double* d_part, double* d_out);
int launch_reconstruct(sdqz_ctx* ctx, const uint16_t* codes, const OutLookup& ol,
                       const uint8_t* blockflag, bool any_slow, int ndims, const uint64_t dims[3],
                       const uint32_t block[3], uint32_t cap, double two_eb, void* out,
                       int out_kind);

// helpers
__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
uint32_t default_chunk_size(uint64_t n);
bool is_fast_shape(int ndims, const uint32_t block[3]);
bool env_disabled(const char* name);   // env var set and not "0"

}  // namespace sdqz
