/*
 * sdqz_cuda.h -- C-ABI of libsdqz_cuda.so, the B200 (sm_100a) implementation of
 * the sdqz compression path (cuSZ dual-quantization + canonical Huffman).
 *
 * The reference (`sdqz`, /root/reference/pkg/src/sdqz) is pure Python; its
 * "plugin interface" for this path is the set of stage functions composed in
 * pipeline.py.  Each entry point below replaces one of them (cited as
 * reference file:line); the Python package paper_2007_09625_b200 binds them
 * with ctypes and keeps the reference's names, argument meaning and error
 * classes.  No torch types cross this boundary: plain pointers and sizes.
 *
 * Conventions
 *   - Every function returns an sdqz_status; on failure the message is
 *     available from sdqz_last_error(ctx).  Codes map to the reference's
 *     exception classes: SDQZ_EINVAL -> SdqzError, SDQZ_ECORRUPT ->
 *     CorruptionError, SDQZ_EFORMAT -> ArchiveFormatError (archive.py:44).
 *   - Pointers named d_* are device pointers owned by the caller; h_* are host
 *     pointers.  Scratch memory is owned by the context and reused.
 *   - Calls are stream-ordered on the context's stream.  Functions returning
 *     sizes or errors synchronize that stream before returning.
 *   - dtype codes: 0 = float32, 1 = float64 (archive.py:38).
 *   - dims/block arrays always have 3 entries; unused trailing entries are 1
 *     (archive.py:15).
 */
#ifndef SDQZ_CUDA_H
#define SDQZ_CUDA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SDQZ_API __attribute__((visibility("default")))
#else
#define SDQZ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SDQZ_OK = 0,
    SDQZ_EINVAL = 1,   /* SdqzError            (core.py:26)    */
    SDQZ_ECORRUPT = 2, /* CorruptionError      (core.py:30)    */
    SDQZ_EFORMAT = 3,  /* ArchiveFormatError   (archive.py:44) */
    SDQZ_ECUDA = 4,    /* CUDA runtime failure                 */
} sdqz_status;

typedef struct sdqz_ctx sdqz_ctx;

/* Header fields of one archive (archive.py:3-13, struct "<4s4B3Q2d5IB3Q"). */
typedef struct {
    uint8_t dtype_code;      /* 0 f32, 1 f64                     */
    uint8_t ndims;           /* 1..3                             */
    uint8_t eb_mode;         /* 0 abs, 1 valrel                  */
    uint8_t unit_width;      /* 32 | 64                          */
    uint64_t dims[3];
    double eb_resolved;
    double eb_specified;
    uint32_t cap;
    uint32_t block[3];
    uint32_t chunk_size;
    uint64_t n_outliers;
    uint64_t n_chunks;
    uint64_t payload_bytes;
} sdqz_header;

#define SDQZ_HEADER_SIZE 93

/* ---- context ------------------------------------------------------------ */
/* stream: a cudaStream_t (NULL = create a private non-blocking stream). */
SDQZ_API int sdqz_ctx_create(int device, void* stream, sdqz_ctx** out);
SDQZ_API int sdqz_ctx_destroy(sdqz_ctx* ctx);
SDQZ_API int sdqz_ctx_set_stream(sdqz_ctx* ctx, void* stream);
SDQZ_API const char* sdqz_last_error(const sdqz_ctx* ctx);
/* Total kernels launched through this context (evidence for the bench). */
SDQZ_API uint64_t sdqz_kernel_launches(const sdqz_ctx* ctx);
/* Compress / decompress calls served by replaying a captured CUDA graph (a
 * call repeating the previous call's pointers and parameters is captured once,
 * then replayed; disabled while the kernel timer runs or SDQZ_NO_GRAPH=1). */
SDQZ_API uint64_t sdqz_graph_replays(const sdqz_ctx* ctx);
/* Per-kernel device timer: on=1 resets and starts accumulating CUDA-event
 * intervals per kernel name on the context's stream; sdqz_kernel_times writes
 * "name=ms;name=ms;..." (NUL-terminated, truncated to len) and returns the
 * untruncated length. */
SDQZ_API int sdqz_set_timing(sdqz_ctx* ctx, int on);
/* Diagnostics of the last call (inflate: lane redecodes, unsynchronised
 * chunks, chunks decoded by the sequential path). */
SDQZ_API int sdqz_debug_counters(sdqz_ctx* ctx, uint64_t* out, int n);
/* Copy `bytes` of context scratch slot `slot` to host (diagnostics only). */
SDQZ_API int sdqz_debug_read(sdqz_ctx* ctx, int slot, void* host, uint64_t bytes);
SDQZ_API int sdqz_kernel_times(sdqz_ctx* ctx, char* buf, uint64_t len);

/* ---- L1: field description (core.py:136-175) ---------------------------- */
/* min/max in the input dtype (returned widened to double) + nonfinite flag. */
SDQZ_API int sdqz_describe(sdqz_ctx* ctx, const void* d_in, int dtype, uint64_t n,
                  double* vmin, double* vmax, int* nonfinite);

/* Host -> device copy of a pageable host buffer through the context's pinned
 * staging (parallel host copy overlapped with the DMA); synchronous. */
SDQZ_API int sdqz_upload(sdqz_ctx* ctx, const void* h_src, uint64_t bytes, void* d_dst);

/* Reconstruction quality (metrics.py:52-76) in one fp64 pass over both
 * device arrays: out = {sum (a-b)^2, max |a-b|, min a, max a, nonfinite(a)}.
 * Replaces the reference's numpy reductions in quality() / rd_sweep(). */
SDQZ_API int sdqz_quality(sdqz_ctx* ctx, const void* d_orig, int orig_dtype, const void* d_recon,
                          int recon_dtype, uint64_t n, double* out);

/* ---- L2 lossy stage (dualquant.py) --------------------------------------- */
/* prequantize (dualquant.py:62-78): d_out[i] = copysign(floor(|x/(2eb)|+.5), x/(2eb)). */
SDQZ_API int sdqz_prequantize(sdqz_ctx* ctx, const void* d_in, int dtype, uint64_t n, double eb,
                     double* d_out);

/* compress_field codes (dualquant.py:172-194, :242-273): writes one uint16 code per
 * point (0 = outlier) and, if d_hist != NULL, the exact histogram (uint64[cap],
 * overwritten).  in_kind: 0 f32 data, 1 f64 data, 2 f64 already-prequantized
 * units (postquantize_block, dualquant.py:132-147).  *nonfinite is set when an
 * input value is NaN/Inf. */
SDQZ_API int sdqz_dualquant(sdqz_ctx* ctx, const void* d_in, int in_kind, int ndims,
                   const uint64_t dims[3], const uint32_t block[3], double eb, uint32_t cap,
                   uint16_t* d_codes, uint64_t* d_hist, int* nonfinite);

/* Outlier list of a code array (dualquant.py:190-194): records {uint64 flat index,
 * fp64 prequantized value} for every code 0, ascending row-major, the value
 * recomputed from the input.  Capacity max_k records; *k_out = number found. */
SDQZ_API int sdqz_outliers(sdqz_ctx* ctx, const void* d_in, int in_kind, const uint16_t* d_codes,
                  uint64_t n, double eb, void* d_records, uint64_t max_k, uint64_t* k_out);

/* reconstruct_field (dualquant.py:276-332): validates like _validate_output and
 * writes flat values: out_kind 0 -> float32(x*2eb), 1 -> float64 x*2eb.
 * code_bytes: 2 (uint16 codes) or 4 (uint32 codes, range-checked against cap). */
SDQZ_API int sdqz_reconstruct(sdqz_ctx* ctx, const void* d_codes, int code_bytes, uint64_t n,
                     const uint64_t* d_idx, const double* d_val, uint64_t k, int ndims,
                     const uint64_t dims[3], const uint32_t block[3], double eb, uint32_t cap,
                     void* d_out, int out_kind);

/* ---- L2 lossless stage (huffman.py) ------------------------------------- */
/* histogram (huffman.py:77-95) over uint32 codes; counts uint64[cap]. */
SDQZ_API int sdqz_histogram_u32(sdqz_ctx* ctx, const uint32_t* d_codes, uint64_t n, uint32_t cap,
                       uint64_t* d_hist);

/* build_tree (huffman.py:98-131) -> bitwidth per symbol (uint8[cap]). */
SDQZ_API int sdqz_build_tree(sdqz_ctx* ctx, const uint64_t* d_hist, uint32_t cap, uint8_t* d_bw);

/* canonize (huffman.py:146-190).  d_entries: uint64[cap] packed units (a 32-bit
 * unit is stored zero-extended).  Reverse tables: d_first uint64[58],
 * d_offsets int64[59], d_symbols uint32[cap]; *n_present symbols valid. */
SDQZ_API int sdqz_canonize(sdqz_ctx* ctx, const uint8_t* d_bw, uint32_t cap, uint64_t* d_entries,
                  uint64_t* d_first, int64_t* d_offsets, uint32_t* d_symbols,
                  int* unit_width, int* max_bw, uint32_t* n_present);

/* encode (huffman.py:193-203): d_units (uint32 or uint64 per unit_width). */
SDQZ_API int sdqz_encode_u32(sdqz_ctx* ctx, const uint32_t* d_codes, uint64_t n, const uint64_t* d_entries,
                    uint32_t cap, int unit_width, void* d_units);

/* deflate (huffman.py:219-269) of packed units.  d_payload capacity
 * payload_cap bytes; *payload_bytes = used.  chunk bit lengths uint32[C]. */
SDQZ_API int sdqz_deflate_units(sdqz_ctx* ctx, const void* d_units, int unit_width, uint64_t n,
                       uint32_t chunk, uint32_t* d_chunk_bits, uint8_t* d_payload,
                       uint64_t payload_cap, uint64_t* payload_bytes);

/* encode + deflate (huffman.py:193-269) of uint16 codes with a packed codebook
 * (d_entries uint64[cap] from sdqz_canonize): the fused path's K4 without the
 * outlier compaction.  Used per shard by the multi-GPU compress. */
SDQZ_API int sdqz_encode_deflate(sdqz_ctx* ctx, const uint16_t* d_codes, uint64_t n,
                        const uint64_t* d_entries, uint32_t cap, uint32_t chunk,
                        uint32_t* d_chunk_bits, uint8_t* d_payload, uint64_t payload_cap,
                        uint64_t* payload_bytes);

/* inflate (huffman.py:311-356) with the canonical reverse tables. */
SDQZ_API int sdqz_inflate(sdqz_ctx* ctx, const uint8_t* d_payload, uint64_t payload_bytes,
                 const uint32_t* d_chunk_bits, uint64_t n_chunks, uint32_t chunk,
                 const uint64_t* d_first, const int64_t* d_offsets, const uint32_t* d_symbols,
                 int max_bw, uint64_t n, uint32_t* d_codes_u32);

/* ---- L4 fused pipeline (pipeline.py:15-58) ------------------------------- */
/* compress (pipeline.py:15-39) of a device-resident field.  eb_mode 0 abs,
 * 1 valrel; chunk 0 = default_chunk_size(n).  On success *hdr describes the
 * archive, whose sections stay in context memory until the next compress. */
SDQZ_API int sdqz_compress(sdqz_ctx* ctx, const void* d_in, int dtype, int ndims, const uint64_t dims[3],
                  const uint32_t block[3], int eb_mode, double eb, uint32_t cap, uint32_t chunk,
                  sdqz_header* hdr);
/* sdqz_compress with the field's K1 result supplied: stats = {vmin, vmax,
 * nonfinite} as returned by sdqz_describe of the same (unchanged) field; the
 * describe pass is skipped.  rd_sweep reuses one describe across its bounds
 * (metrics.py:89-118). */
SDQZ_API int sdqz_compress_described(sdqz_ctx* ctx, const void* d_in, int dtype, int ndims,
                                     const uint64_t dims[3], const uint32_t block[3], int eb_mode, double eb,
                                     uint32_t cap, uint32_t chunk, const double stats[3], sdqz_header* hdr);
/* Total archive bytes of the last compress. */
SDQZ_API uint64_t sdqz_archive_size(const sdqz_ctx* ctx);
/* Id of the last compress's archive (unique per process; 0 = none, e.g. after
 * a call that reused the section buffers).  A device-archive handle records it
 * and passes it to the two calls below, which reject a stale id with
 * SDQZ_EINVAL instead of returning another archive's sections. */
SDQZ_API uint64_t sdqz_archive_generation(const sdqz_ctx* ctx);
/* Write archive `gen` (header + sections) to host memory (gen 0: the last). */
SDQZ_API int sdqz_archive_write(sdqz_ctx* ctx, uint64_t gen, uint8_t* h_dst, uint64_t capacity);
/* Copy archive `gen`'s sections into caller device buffers (stream-ordered,
 * no sync; any pointer may be NULL to skip that section). */
SDQZ_API int sdqz_archive_copy(sdqz_ctx* ctx, uint64_t gen, uint8_t* d_bw, void* d_outliers,
                               uint32_t* d_chunk_bits, uint8_t* d_payload);
/* Device pointers to archive `gen`'s sections (bitwidths, outlier records,
 * chunk bits, payload) -- for device-resident decompress and sharding. */
SDQZ_API int sdqz_archive_sections(sdqz_ctx* ctx, uint64_t gen, const uint8_t** d_bw, const void** d_outliers,
                          const uint32_t** d_chunk_bits, const uint8_t** d_payload);

/* ---- sharded compress (one rank, one slab of whole block rows)
 * The reference composes the same slab decomposition for workers > 1
 * (dualquant.py:230-273); these phases wrap the per-slab pipeline around the
 * caller's collectives:
 *   describe -> [all-reduce MAX of d_range] -> quantize -> [all-reduce SUM of
 *   d_hist] -> (head/tail code exchange if chunks straddle slabs) -> encode.
 * Nothing reaches the host before encode's sizes.  After encode the rank's
 * sections (bitwidths, its outlier records with GLOBAL indices, its chunk
 * bits, its payload) are this context's archive (sdqz_archive_sections). */
typedef struct {
    uint64_t n_chunks;       /* chunks this rank packed                   */
    uint64_t payload_bytes;  /* their payload bytes                       */
    uint64_t n_outliers;     /* this slab's outlier records               */
    uint32_t unit_width;     /* 32 | 64 (global codebook: same everywhere) */
    uint32_t max_bw;
    double eb_resolved;      /* same everywhere (core.py:161-175)         */
} sdqz_shard_sizes;
/* describe (core.py:136-158) of this slab into d_range[3] = {-min, max,
 * nonfinite} (device doubles) for an all-reduce MAX.  No host sync. */
SDQZ_API int sdqz_shard_describe(sdqz_ctx* ctx, const void* d_in, int dtype, uint64_t n, double* d_range);
/* resolve the bound from the reduced range (valrel) or eb (abs) on device,
 * dual-quant the slab (local dims) into the context's code buffer and its
 * histogram into d_hist (u64[cap], device) for an all-reduce SUM.  No sync. */
SDQZ_API int sdqz_shard_quantize(sdqz_ctx* ctx, const void* d_in, int dtype, int ndims, const uint64_t dims[3],
                                 const uint32_t block[3], int eb_mode, double eb, uint32_t cap,
                                 const double* d_range, uint64_t* d_hist);
/* copy the slab's first `count` codes (its head, packed by the previous rank
 * when chunks straddle the slab start) to d_dst. */
SDQZ_API int sdqz_shard_head(sdqz_ctx* ctx, uint64_t count, uint16_t* d_dst);
/* codebook from the global histogram (huffman.py:98-190), deflate
 * (huffman.py:219-269) of codes [head, n) + the next ranks' n_tail head codes
 * in chunks of `chunk`, outlier records (dualquant.py:190-194) of all n slab
 * points with global index idx_base + local.  Synchronous; checks in the
 * reference's order (resolve_error_bound first). */
SDQZ_API int sdqz_shard_encode(sdqz_ctx* ctx, const uint64_t* d_hist, uint32_t chunk, uint64_t head,
                               const uint16_t* d_tail, uint64_t n_tail, uint64_t idx_base,
                               sdqz_shard_sizes* out);

/* parse_header (archive.py:143-181): validate and decode the 93-byte header. */
SDQZ_API int sdqz_parse_header(sdqz_ctx* ctx, const uint8_t* h_buf, uint64_t len, sdqz_header* hdr);

/* decompress (pipeline.py:42-58 + archive.deserialize :184-246) of a host
 * archive into device memory (d_out: float32/float64 per header dtype). */
SDQZ_API int sdqz_decompress(sdqz_ctx* ctx, const uint8_t* h_archive, uint64_t len, void* d_out);

/* decompress from device-resident sections (same checks as deserialize). */
/* decompress_sections + quality (metrics.py:52-76) against the original
 * device field d_orig, the reduction fused into the reconstruct kernels'
 * epilogue (one pass: codes + original in, field out).  q5 as sdqz_quality.
 * *fused = 0 when the path had no fused kernel (generic block shapes, blocks
 * replayed in fp64); the scores then come from a separate pass.  Used by
 * rd_sweep / the CLI sweep (metrics.py:89-118). */
SDQZ_API int sdqz_decompress_quality(sdqz_ctx* ctx, const sdqz_header* hdr, const uint8_t* d_bw,
                                     const void* d_outliers, const uint32_t* d_chunk_bits,
                                     const uint8_t* d_payload, void* d_out, const void* d_orig, int orig_dtype,
                                     double* q5, int* fused);

/* ---- host-buffer pipeline (no caller-side device memory) ----------------
 * The same compress / decompress / quality with HOST input and output
 * buffers: inputs go through the context's pinned staging into context-owned
 * device memory, outputs come back the same way.  For callers without a
 * device allocator (the CLI: python -m paper_2007_09625_b200, cli.py:68-109). */
SDQZ_API int sdqz_device_count(int* n);
/* compress (pipeline.py:15-39) of a host field; archive via sdqz_archive_write. */
SDQZ_API int sdqz_compress_host(sdqz_ctx* ctx, const void* h_in, int dtype, int ndims, const uint64_t dims[3],
                                const uint32_t block[3], int eb_mode, double eb, uint32_t cap, uint32_t chunk,
                                sdqz_header* hdr);
/* decompress (pipeline.py:56-58) of a host archive into host memory
 * (float32/float64 per header dtype, dims[0]*dims[1]*dims[2] values). */
SDQZ_API int sdqz_decompress_host(sdqz_ctx* ctx, const uint8_t* h_archive, uint64_t len, void* h_out);
/* quality (metrics.py:52-76) of two host arrays (out as sdqz_quality). */
SDQZ_API int sdqz_quality_host(sdqz_ctx* ctx, const void* h_orig, int orig_dtype, const void* h_recon,
                               int recon_dtype, uint64_t n, double* out);

SDQZ_API int sdqz_decompress_sections(sdqz_ctx* ctx, const sdqz_header* hdr, const uint8_t* d_bw,
                             const void* d_outliers, const uint32_t* d_chunk_bits,
                             const uint8_t* d_payload, void* d_out);

/* Multi-GPU slab decompress: inflate the chunk range
 * [c0, c0 + n_chunks) covering this rank's slab (device sections: the range's
 * chunk bit lengths and payload bytes, zero padded by >= 64 bytes), then
 * reconstruct the slab whose first code is `lo` codes into the range, with
 * the slab's outlier records (ascending; index - idx_base is slab-local, so
 * the records of a sharded archive are used as they are with idx_base = the
 * slab's first point).  Checks as decompress for the slab: decode errors,
 * record range/order, codes[idx] == 0, zero-code count of the slab.
 * Replaces the per-rank pipeline.py:42-58. */
SDQZ_API int sdqz_decompress_slab(sdqz_ctx* ctx, const sdqz_header* hdr, const uint8_t* d_bw,
                                  const void* d_rec, uint64_t k, uint64_t idx_base,
                                  const uint32_t* d_chunk_bits, uint64_t n_chunks, const uint8_t* d_payload,
                                  uint64_t payload_bytes, uint64_t n_range, uint64_t lo,
                                  const uint64_t local_dims[3], void* d_out);

#ifdef __cplusplus
}
#endif
#endif /* SDQZ_CUDA_H */
