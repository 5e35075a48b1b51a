/*
 * endor_cuda.h -- C ABI of the B200-native Endor decompression path.
 *
 * The reference (arXiv 2406.11674 "Endor", /root/reference/proj) is a
 * header-only C++20 library; its hot path is the CPU scalar decompress.  This
 * header is the drop-in boundary that replaces that path with sm_100a kernels:
 * plain C, plain pointers and sizes, no CUDA or torch types (streams are
 * passed as `void*` holding a cudaStream_t; NULL = legacy default stream).
 * include/endor_cuda.hpp wraps it in the reference's own C++ signatures
 * (endor::cuda::decompress(const EndorTensor&) -> DenseMatrix, ...), and
 * INTEGRATION.md shows the binding a maintainer adds to the reference tree.
 *
 * Reference interfaces replaced (paths under proj/include/endor/):
 *   endor_cuda_decompress            <- decompress             codec.hpp:157-166
 *   endor_cuda_decompress_chunked    <- decompress_chunked     codec.hpp:205-216
 *   endor_cuda_decompress_chunk_into <- decompress_chunk_into  codec.hpp:191-201
 *   endor_cuda_rank_index            <- build_rank_index       bitmap.hpp:117-132
 *   endor_cuda_popcount              <- Bitmap::count          bitmap.hpp:34-38
 *   endor_cuda_compress              <- compress               codec.hpp:97-126
 *   endor_cuda_synth_weight          <- synth_weight           weight_gen.hpp:40-55
 *   endor_cuda_magnitude_prune       <- magnitude_prune        weight_gen.hpp:96-113
 *   endor_cuda_gemv                  <- (absent; the consumer is modelled as a
 *                                        constant compute time, sim.hpp:227)
 *   endor_cuda_gemm_compressed       <- (absent; prefill / batched consumer,
 *                                        sim.hpp:30,256: fused tcgen05 GEMM)
 *   endor_pipeline_*                 <- the Endor offload stages, modelled
 *                                        only analytically at sim.hpp:196-224
 *   endor_cuda_decompress_host       <- decompress() end to end over host
 *                                        buffers (H2D -> kernels -> D2H)
 *
 * Errors.  Every entry point returns an endor_status that maps 1:1 onto the
 * reference's exception classes (error.hpp:9-63) so the C++ wrapper can
 * rethrow the same types.  Host-checkable conditions are returned
 * synchronously.  Conditions only the device can see (bitmap popcount !=
 * nnz, codec.hpp:158-160; rank index inconsistent with the bitmap,
 * codec.hpp:170-184; nonzero bitmap padding bits, bitmap.hpp:78-84) are
 * latched in the workspace and returned by endor_cuda_sync_status(); the
 * kernels that follow a latched error write nothing.
 *
 * Memory.  Device pointers unless a name says _host.  bitmap: ceil(n/8)
 * LSB-first bytes (bit i = byte i>>3, bit i&7; bitmap.hpp:14-17), 4-byte
 * aligned.  values: nnz*elem_bytes raw little-endian elements in row-major
 * order, any alignment.  dense output: 16-byte aligned.  The workspace is
 * caller-owned device memory of endor_cuda_workspace_bytes() bytes; it must be
 * zero-filled once before first use (endor_cuda_workspace_init) and is left
 * zeroed by every successful call.  One workspace per in-flight stream.
 * Nothing on the hot path allocates.
 *
 * Threading.  All entry points are reentrant per (stream, workspace) pair;
 * like the reference inputs are never mutated.
 */
#ifndef ENDOR_CUDA_H
#define ENDOR_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ENDOR_CUDA_ABI_VERSION 4

typedef enum endor_status {
    ENDOR_OK = 0,
    ENDOR_ERR_SIZE = 1,             /* SizeError        error.hpp:15-18  */
    ENDOR_ERR_CORRUPTION = 2,       /* CorruptionError  error.hpp:22-25  */
    ENDOR_ERR_BOUNDS = 3,           /* BoundsError      error.hpp:28-31  */
    ENDOR_ERR_INVALID_ARGUMENT = 4, /* std::invalid_argument             */
    ENDOR_ERR_CUDA = 5,             /* CUDA runtime failure (no reference analogue) */
    ENDOR_ERR_CONFIG = 6,           /* ConfigError      error.hpp:34-37  */
    ENDOR_ERR_FORMAT = 7,           /* FormatError      error.hpp:42-60; kind: endor_cuda_last_format_kind() */
    ENDOR_ERR_IO = 8                /* Error("cannot open ..." / "short read ...") file_io.hpp:159-172 */
} endor_status;

/* FormatError::Kind (error.hpp:45-52) */
typedef enum endor_format_kind {
    ENDOR_FMT_TRUNCATED = 0,
    ENDOR_FMT_BAD_MAGIC = 1,
    ENDOR_FMT_BAD_VERSION = 2,
    ENDOR_FMT_BAD_CRC = 3,
    ENDOR_FMT_COUNT_MISMATCH = 4,
    ENDOR_FMT_MALFORMED = 5
} endor_format_kind;

/* Dtype codes, dense_matrix.hpp:18-21 (also the on-disk codes). */
#define ENDOR_DTYPE_F16 0
#define ENDOR_DTYPE_I8 1

/* Device-side view of an EndorTensor (codec.hpp:24-66). */
typedef struct endor_tensor_view {
    uint64_t rows;
    uint64_t cols;
    int32_t dtype;       /* ENDOR_DTYPE_* */
    int32_t reserved;
    const void* bitmap;  /* ceil(rows*cols/8) bytes, 4-byte aligned */
    const void* values;  /* nnz * elem_bytes bytes */
    uint64_t nnz;
} endor_tensor_view;

/* ---- library ------------------------------------------------------------ */
int endor_cuda_abi_version(void);
const char* endor_cuda_last_error_string(void); /* thread-local detail of the last failure */
const char* endor_cuda_status_name(int status);

/* Elements per expand tile (the kernel's natural unit, a multiple of every
 * RankIndex chunk size <= it). */
uint64_t endor_cuda_tile_elems(void);

/* Workspace for any call on a tensor of up to n = rows*cols elements. */
size_t endor_cuda_workspace_bytes(uint64_t rows, uint64_t cols);
int endor_cuda_workspace_init(void* ws, size_t ws_bytes, void* stream);

/* Wait for `stream` and return (and clear) any device-latched status. */
int endor_cuda_sync_status(void* ws, void* stream);

/* ---- hot path ----------------------------------------------------------- */

/* decompress (codec.hpp:157-166): dense_out[n*eb] <- t.  Asynchronous. */
int endor_cuda_decompress(const endor_tensor_view* t, void* dense_out, void* ws, size_t ws_bytes,
                          void* stream);

/* decompress of up to 64 tensors of one dtype in two launches total (one
 * count, one persistent expand over all of their tiles) -- e.g. every weight
 * matrix of a decoder layer.  Bitmaps and outputs 16-byte aligned; the
 * workspace needs endor_cuda_workspace_bytes_batch(views, count) bytes.
 * Same results and errors as endor_cuda_decompress on each tensor. */
size_t endor_cuda_workspace_bytes_batch(const endor_tensor_view* views, int count);
int endor_cuda_decompress_batch(const endor_tensor_view* views, void* const* dense_outs, int count,
                                void* ws, size_t ws_bytes, void* stream);
/* The same split into its launches (phase 1 = count, 2 = expand, 0 = both),
 * for per-kernel timing. */
int endor_cuda_decompress_batch_phase(const endor_tensor_view* views, void* const* dense_outs,
                                      int count, int phase, void* ws, size_t ws_bytes, void* stream);

/* decompress(dequantize_values(t)) fused (codec.hpp:334-349 then :157): t is
 * an I8 tensor (ENDOR_DTYPE_I8) quantized with `scale` (quantize_values,
 * codec.hpp:306-331); dense_f16_out receives n f16 elements, each set one
 * f32_to_f16(float(q) * scale) bit-exactly (float16.hpp:35-73), unset +0.
 * Reads 1/8 + (1-s) bytes per element instead of 1/8 + 2(1-s). */
int endor_cuda_decompress_dequant(const endor_tensor_view* t, float scale, void* dense_f16_out, void* ws,
                                  size_t ws_bytes, void* stream);

/* Selective decompression (activation sparsity):
 *   extract_rows (codec.hpp:239-266): out[nsel, cols] = dense rows rows_dev[..]
 *   extract_cols (codec.hpp:271-297): out[rows, nsel] = dense columns cols_dev[..]
 * Index lists are device u64 arrays, sorted and unique (check_sorted_unique,
 * codec.hpp:224-232: out-of-range -> BOUNDS, unsorted/duplicate -> INVALID,
 * first failing position wins; device-latched).  Bitmap 16-byte aligned. */
int endor_cuda_extract_rows(const endor_tensor_view* t, const uint64_t* rows_dev, uint64_t nsel, void* out,
                            void* ws, size_t ws_bytes, void* stream);
int endor_cuda_extract_cols(const endor_tensor_view* t, const uint64_t* cols_dev, uint64_t nsel, void* out,
                            void* ws, size_t ws_bytes, void* stream);

/* endor_cuda_decompress split into its two launches, for per-kernel timing:
 * phase 1 = rank (count) kernel, phase 2 = expand kernel (needs phase 1 on
 * the same workspace first).  phase 1 then 2 == endor_cuda_decompress. */
int endor_cuda_decompress_phase(const endor_tensor_view* t, void* dense_out, int phase, void* ws,
                                size_t ws_bytes, void* stream);

/* build_rank_index (bitmap.hpp:117-132) on device: prefix_out[ceil(n/cs)]
 * u64 exclusive per-chunk popcounts.  cs must be a power of two >= 64, else
 * ENDOR_ERR_INVALID_ARGUMENT (bitmap.hpp:118-120).  total_out (device u64,
 * may be NULL) receives the popcount. */
int endor_cuda_rank_index(const void* bitmap, uint64_t n, uint64_t chunk_size, uint64_t* prefix_out,
                          uint64_t* total_out, void* ws, size_t ws_bytes, void* stream);

/* Bitmap::count (bitmap.hpp:34-38) into a device u64. */
int endor_cuda_popcount(const void* bitmap, uint64_t n, uint64_t* total_out, void* ws,
                        size_t ws_bytes, void* stream);

/* decompress_chunked (codec.hpp:205-216) with a device-resident RankIndex.
 * chunk_count must equal ceil(n/cs) (else CORRUPTION, codec.hpp:174-176).
 * Any nonzero chunk size is accepted, as by the reference's RankIndex
 * constructor (bitmap.hpp:104).  cs == 1024: single-launch fast path,
 * check_index semantics (see endor_cuda_decompress_chunked_batch).
 * cs == 2048 / 4096 / 8192 (4096 is the reference's kDefaultChunkSize,
 * codec.hpp:19): also one launch (16-byte aligned bitmap and prefix), the
 * sub-tile starts derived from the bitmap on chip and EVERY entry verified.
 * Other sizes: a counting pass, then every prefix entry is verified on device
 * (a superset of check_index), then the expand. */
int endor_cuda_decompress_chunked(const endor_tensor_view* t, uint64_t chunk_size,
                                  const uint64_t* prefix, uint64_t chunk_count, void* dense_out,
                                  void* ws, size_t ws_bytes, void* stream);

/* decompress_chunked over up to 64 tensors.  With chunk_size == 1024 (the
 * recommended load-time index: 8 bytes per 1024 elements) and 16-byte aligned
 * bitmaps and prefixes, the index supplies every sub-tile's value offset, so
 * the whole batch is ONE expand launch with no counting pass; like the
 * reference's check_index (codec.hpp:170-184) only the last entry is
 * verified (prefix[last] + tail popcount == nnz), and an inconsistent middle
 * entry produces unspecified output (never an out-of-bounds access).  Chunk
 * sizes 2048 / 4096 / 8192 are one launch for the batch too (every entry
 * verified, see endor_cuda_decompress_chunked); other chunk sizes fall back
 * to endor_cuda_decompress_chunked per tensor.
 * prefixes[i] must hold ceil(n_i / chunk_size) entries. */
int endor_cuda_decompress_chunked_batch(const endor_tensor_view* views, const uint64_t* const* prefixes,
                                        uint64_t chunk_size, void* const* dense_outs, int count, void* ws,
                                        size_t ws_bytes, void* stream);

/* decompress_chunk_into (codec.hpp:191-201): writes exactly and only chunk
 * k's byte range of dense_out (which must hold the full dense matrix,
 * dense_out_bytes == n*eb, else INVALID_ARGUMENT; k >= chunk_count ->
 * BOUNDS).  Like check_index, verifies prefix[last] + tail popcount == nnz.
 * Any nonzero chunk size (chunk ranges may start and end inside a bitmap
 * word; the neighbouring elements are never written). */
int endor_cuda_decompress_chunk_into(const endor_tensor_view* t, uint64_t chunk_size,
                                     const uint64_t* prefix, uint64_t chunk_count, uint64_t k,
                                     void* dense_out, uint64_t dense_out_bytes, void* ws,
                                     size_t ws_bytes, void* stream);

/* Same as endor_cuda_decompress over HOST buffers: H2D of bitmap+values,
 * decompress, D2H of the dense matrix, synchronous, device buffers cached
 * per thread.  This is what endor::cuda::decompress(const EndorTensor&) calls. */
int endor_cuda_decompress_host(uint64_t rows, uint64_t cols, int32_t dtype,
                               const void* bitmap_host, const void* values_host, uint64_t nnz,
                               void* dense_host_out);

/* Host-buffer, synchronous forms of the other reference entry points (what
 * the endor::cuda:: C++ wrappers call).  Check order and error codes follow
 * the reference exactly: check_index (CORRUPTION) before the chunk bound
 * (BOUNDS) before the destination size (INVALID_ARGUMENT), codec.hpp:193-197. */
int endor_cuda_rank_index_host(const void* bitmap_host, uint64_t n, uint64_t chunk_size,
                               uint64_t* prefix_host_out);
int endor_cuda_decompress_chunked_host(uint64_t rows, uint64_t cols, int32_t dtype,
                                       const void* bitmap_host, const void* values_host,
                                       uint64_t nnz, uint64_t chunk_size,
                                       const uint64_t* prefix_host, uint64_t chunk_count,
                                       void* dense_host_out);
int endor_cuda_decompress_chunk_into_host(uint64_t rows, uint64_t cols, int32_t dtype,
                                          const void* bitmap_host, const void* values_host,
                                          uint64_t nnz, uint64_t chunk_size,
                                          const uint64_t* prefix_host, uint64_t chunk_count,
                                          uint64_t k, void* dense_host, uint64_t dense_host_bytes);
/* compress over host buffers: values_host_out needs n*eb capacity. */
int endor_cuda_compress_host(uint64_t rows, uint64_t cols, int32_t dtype, const void* dense_host,
                             void* bitmap_host_out, void* values_host_out, uint64_t* nnz_out,
                             int32_t* negzero_out);
/* extract_rows / extract_cols (codec.hpp:239-297) on host buffers (sync):
 * out_host receives nsel*cols (rows) or rows*nsel (cols) elements. */
int endor_cuda_extract_rows_host(uint64_t rows, uint64_t cols, int32_t dtype, const void* bitmap_host,
                                 const void* values_host, uint64_t nnz, const uint64_t* rows_host, uint64_t nsel,
                                 void* out_host);
int endor_cuda_extract_cols_host(uint64_t rows, uint64_t cols, int32_t dtype, const void* bitmap_host,
                                 const void* values_host, uint64_t nnz, const uint64_t* cols_host, uint64_t nsel,
                                 void* out_host);
/* quantize_values / dequantize_values (codec.hpp:306-349) of packed values on
 * host buffers (sync). */
int endor_cuda_quantize_values_host(const void* values_f16_host, uint64_t nnz, void* q_host_out, float* scale_out);
int endor_cuda_dequantize_values_host(const void* q_host, uint64_t nnz, float scale, void* f16_host_out);

/* ---- input producers (offline in the paper) ---------------- */

/* compress (codec.hpp:97-126) on device.  values_out must hold n*eb bytes
 * (worst case); *nnz_out_host and *negzero_out_host are written.  Synchronous. */
int endor_cuda_compress(uint64_t rows, uint64_t cols, int32_t dtype, const void* dense,
                        void* bitmap_out, void* values_out, uint64_t* nnz_out_host,
                        int32_t* negzero_out_host, void* ws, size_t ws_bytes, void* stream);

/* synth_weight (weight_gen.hpp:40-55), bit-exact, for rows [row0, row0+nrows)
 * of a rows x cols matrix (element index i = global row-major index). */
int endor_cuda_synth_weight(uint64_t rows, uint64_t cols, int32_t dtype, uint64_t seed,
                            uint64_t row0, uint64_t nrows, void* out, void* stream);

/* magnitude_prune (weight_gen.hpp:96-113) in place over n elements,
 * bit-exact (exactly floor(s*n) smallest |v| zeroed, ties at the lower index).
 * Synchronous (one small D2H for the threshold). */
int endor_cuda_magnitude_prune(uint64_t n, int32_t dtype, double sparsity, void* w, void* ws,
                               size_t ws_bytes, void* stream);

/* quantize_values (codec.hpp:306-331) on device, bit-exact: symmetric absmax
 * f16 -> i8 over the packed values (the bitmap is unchanged); the scale
 * (absmax/127, 1.0 for all-zero) is returned through scale_out_host.  Sync. */
int endor_cuda_quantize_values(const void* values_f16, uint64_t nnz, void* q_out, float* scale_out_host,
                               void* ws, size_t ws_bytes, void* stream);

/* dequantize_values (codec.hpp:334-349) on device, bit-exact: out_f16[i] =
 * f32_to_f16(float(q[i]) * scale) over the packed values (the bitmap is
 * unchanged; float16.hpp:35-73 RNE, NaN products as on the reference's x86).
 * Async on the stream. */
int endor_cuda_dequantize_values(const void* q_i8, uint64_t nnz, float scale, void* out_f16, void* stream);

/* ---- lossless transport coding of the packed values (no reference counterpart) ----
 * The Endor mode is bound by the host -> GPU link (sim.hpp:200-204, 322-325):
 * every byte of the values section crosses it.  The high byte of a pruned f16
 * weight (sign, exponent, top two mantissa bits) takes few distinct values, the
 * low byte is noise, so the blob keeps the low bytes raw and codes the high
 * byte in k bits (1..7) through a dictionary of the 2^k - 1 most frequent high
 * bytes; code 2^k - 1 marks an exception, listed as (index << 8 | high byte).
 * k minimises the blob per tensor.  Decoding reproduces the values bit for bit.
 * Blob (little-endian; every section 16-byte aligned):
 *   endor_vcode_header (256 B) | lo: nnz low bytes (zero-padded to a multiple
 *   of 32) | codes: ceil(nnz / 32) * k u32 words, value i's code at bits
 *   [k i, k i + k) of the word stream (zero-padded to 16 B) | exc: n_exc u64,
 *   ascending index. */
typedef struct endor_vcode_header {
    uint32_t magic;          /* "EVC1" = 0x31435645 */
    uint32_t k;              /* code bits per value, 1..7 */
    uint64_t nnz;            /* values */
    uint64_t n_exc;          /* exceptions */
    uint64_t lo_off, code_off, exc_off, blob_bytes;  /* section offsets, total size */
    uint8_t reserved[8];
    uint8_t dict[128];       /* high byte of code c (c < 2^k - 1) */
    uint8_t pad[64];
} endor_vcode_header;

/* Encode nnz packed f16 values (host memory) into a blob.  blob_out == NULL:
 * only *blob_bytes is computed (size query).  k_max 1..7: the fixed-width
 * dictionary code above with at most k_max bits; k_max 0: automatic -- that,
 * or a Huffman blob ("EVH1", magic 0x31485645) when smaller: the high bytes
 * as a canonical Huffman stream (codes <= 12 bits, LSB first) in chunks of 512
 * values, each starting on a u32 word.  EVH1 layout: header (k = 12, n_exc =
 * stream words) | 4096 x u16 decode table (symbol | length << 8, indexed by
 * the next 12 stream bits) | lo (nnz, padded to 32) | chunk word offsets (u32
 * x (chunks + 1), padded to 16) | stream (zero-padded to 16 bytes).
 * The blob is not capped at the raw size: ship it only when *blob_bytes < 2 nnz
 * (incompressible high bytes make it larger).  Multi-threaded on the host; an
 * offline, load-time step like compress. */
int endor_values_encode(const void* values_f16, uint64_t nnz, int k_max, void* blob_out, size_t blob_cap,
                        size_t* blob_bytes);
/* Validate a blob header (host copy): magic, k, and offsets recomputed from
 * nnz / k / n_exc.  CORRUPTION when inconsistent. */
int endor_values_decode_host_check(const void* header_host);
/* Decode a device copy of the blob into nnz f16 values (values_out, 16-byte
 * aligned); header_host is a host copy of its header (for the launch shape).
 * Two launches (decode, exception patch), async on the stream. */
int endor_cuda_values_decode(const void* header_host, const void* blob_dev, void* values_out, void* stream);

/* ---- consumer ------------------------------------------------------------ */

/* y[rows] = W[rows, cols] . x[cols]; f16 W and x, fp32 accumulate.  y_f32
 * and/or y_f16 may be NULL.  W rows are outputs (catalog orientation). */
int endor_cuda_gemv(uint64_t rows, uint64_t cols, const void* w_f16, const void* x_f16,
                    float* y_f32, void* y_f16, void* stream);

/* Batched dense GEMV: y_i = W_i x_i for up to 64 matrices (one decoder
 * layer) in one launch.  y_f32 / y_f16 arrays (and their entries) may be
 * NULL, not both for a matrix.  Same numerics as endor_cuda_gemv. */
int endor_cuda_gemv_batch(const uint64_t* rows, const uint64_t* cols, const void* const* w_f16,
                          const void* const* x_f16, float* const* y_f32, void* const* y_f16, int count,
                          void* stream);

/* Fused decompress -> GEMV: y = W x straight from the
 * compressed W (bitmap + packed values) -- the dense W is never written, so
 * HBM traffic is 1/8 + 2(1-s) bytes per weight instead of decompress (write
 * 2) + GEMV (read 2).  f16 W with cols % 1024 == 0 (each 1024-element
 * sub-tile is one row segment), x 16-byte aligned, fp32 accumulation; y_f32
 * and/or y_f16.  prefix1024 (optional, device): the tensor's RankIndex at
 * chunk 1024 -- when given no counting pass runs.  Deterministic: each row
 * sums its cols/1024 sub-tile partials in order. */
int endor_cuda_gemv_compressed(const endor_tensor_view* t, const uint64_t* prefix1024, const void* x_f16,
                               float* y_f32, void* y_f16, void* ws, size_t ws_bytes, void* stream);

/* Batched fused decompress -> GEMV: y_i = W_i x_i for up to 64 tensors (one
 * decoder layer's ops) in one persistent launch (+ one counting launch when
 * some prefix1024[i] is NULL, + one row-sum launch).  prefixes1024 may be
 * NULL (count every tensor); y_f32 / y_f16 arrays may be NULL, entries too.
 * Workspace: endor_cuda_workspace_bytes_batch(views, count). */
int endor_cuda_gemv_compressed_batch(const endor_tensor_view* views, const uint64_t* const* prefixes1024,
                                     const void* const* x_f16, float* const* y_f32, void* const* y_f16,
                                     int count, void* ws, size_t ws_bytes, void* stream);

/* Fused decompress -> GEMM on the tcgen05 tensor cores (north star (b): the
 * prefill / batched-decode consumer; the reference models it only as a
 * constant, sim.hpp:30,256):  Y[t, r] = sum_c W[r, c] X[t, c]  for t < tokens,
 * i.e. Y = X W^T with W the decompressed tensor (codec.hpp:157) -- which is
 * never written to HBM: each CTA expands its 128-row W tile into shared
 * memory as the MMA's A operand.  f16 W (any rows / cols), X f16
 * [tokens][x_ld] row-major (16-byte aligned, x_ld >= cols, x_ld % 8 == 0),
 * fp32 accumulation; Y [tokens][rows] as y_f32 and/or y_f16.  prefix1024
 * (optional, device): the tensor's RankIndex at chunk 1024 -- when given no
 * counting pass runs.  Errors as decompress (popcount != nnz, padding bits,
 * an inconsistent index: CorruptionError via endor_cuda_sync_status).
 * Deterministic (split-K partials are summed in a fixed order).  Workspace:
 * endor_cuda_gemm_workspace_bytes(rows, cols, tokens). */
size_t endor_cuda_gemm_workspace_bytes(uint64_t rows, uint64_t cols, uint64_t tokens);
/* (Above ENDOR_GEMM_TWO_PASS_TOKENS tokens, default 384, gemm_compressed
 * decompresses W once into the workspace -- included in the size above -- and
 * runs the dense GEMM below: the fused kernel would re-expand each W tile once
 * per 256-token tile.) */

/* Dense GEMM consumer on tcgen05 (no cuBLAS): Y[t, r] = sum_c W[r, c] X[t, c]
 * with W a dense f16 [rows][cols] (16-byte aligned, cols % 8 == 0), X as in
 * endor_cuda_gemm_compressed, fp32 accumulation, Y [tokens][rows] as y_f32
 * and/or y_f16.  Workspace: endor_cuda_gemm_workspace_bytes(rows, cols,
 * tokens) bytes (split-K partials; zero-initialised once). */
int endor_cuda_gemm(uint64_t rows, uint64_t cols, const void* w_f16, const void* x_f16, uint64_t tokens,
                    uint64_t x_ld, float* y_f32, void* y_f16, void* ws, size_t ws_bytes, void* stream);
int endor_cuda_gemm_compressed(const endor_tensor_view* t, const uint64_t* prefix1024, const void* x_f16,
                               uint64_t tokens, uint64_t x_ld, float* y_f32, void* y_f16, void* ws, size_t ws_bytes,
                               void* stream);

/* ---- storage: .endor containers straight to the GPU ---- */
/* The EndorDirect mode (SsdToGpu, sim.hpp:205-214), executed
 * for real.  Replaces read_endor_file / decode_endor (file_io.hpp:212-277)
 * for a device-resident result: the bitmap and values sections land in
 * caller-owned device buffers. */

typedef struct endor_file_info {
    uint64_t rows, cols, nnz;
    int32_t dtype, flags;          /* flags bit0 quantized, bit1 negative-zero collapsed, bit2 coded values (v3) */
    float quant_scale;             /* flags bit0 */
    uint32_t crc;                  /* stored CRC-32 (IEEE, zlib) of every preceding byte */
    uint32_t header_crc;           /* CRC-32 of the header bytes alone */
    uint32_t gap_bytes;            /* v2: zero fill between the bitmap and values sections */
    uint64_t header_bytes, bitmap_offset, bitmap_bytes, values_offset, values_bytes, file_bytes;
    uint64_t values_out_bytes;     /* bytes endor_reader_read writes to values_dev: nnz * elem bytes
                                      (= values_bytes, except v3: the decoded values, not the blob) */
} endor_file_info;

/* Parse and validate the header and the declared layout in decode_endor's
 * order (magic, version, dtype, flags, fields, rows*cols, nnz, size:
 * file_io.hpp:212-252).  ENDOR_ERR_FORMAT + endor_cuda_last_format_kind().
 * Accepts version 1 (the reference's layout) and version 2 (endor_file_encode_v2:
 * the same fields with the bitmap at byte 4096 and the values at the next 4 KiB
 * boundary, zero fill in between, CRC-32 over every preceding byte -- aligned
 * file offsets, which a GPUDirect Storage DMA needs; nonzero fill is Malformed). */
/* v3 container (no reference counterpart): the v2 layout with flags bit 2 set
 * and the values section holding a coded-values blob of the f16 values
 * (endor_values_encode; not quantized): fewer bytes leave storage, and
 * endor_reader_read decodes them on the GPU after the CRC / padding / popcount
 * checks, so values_dev must hold nnz * 2 bytes (values_out_bytes).
 * endor_file_probe reports the blob's length as values_bytes.  Returns the container size (0 on a bad
 * argument or a blob that does not hold nnz values). */
size_t endor_file_encode_v3(uint64_t rows, uint64_t cols, int32_t flags, const void* bitmap, const void* blob,
                            uint64_t nnz, void* out, size_t out_cap);
int endor_file_probe(const char* path, endor_file_info* out);
int endor_cuda_last_format_kind(void);

/* encode_endor (file_io.hpp:187-210), byte-identical: returns the container
 * size (out == NULL: just the size; 0 on bad arguments / short out_cap). */
size_t endor_file_encode(uint64_t rows, uint64_t cols, int32_t dtype, int32_t flags, float quant_scale,
                         const void* bitmap, const void* values, uint64_t nnz, void* out, size_t out_cap);
/* The version-2 (4 KiB-aligned sections) container of the same tensor; an
 * extension the reference does not read (its decode_endor accepts version 1). */
size_t endor_file_encode_v2(uint64_t rows, uint64_t cols, int32_t dtype, int32_t flags, float quant_scale,
                            const void* bitmap, const void* values, uint64_t nnz, void* out, size_t out_cap);

#define ENDOR_IO_AUTO 0          /* GDS if nvidia-fs is loaded, else POSIX */
#define ENDOR_IO_GDS 1           /* cuFile with nvidia-fs: NVMe -> HBM DMA */
#define ENDOR_IO_CUFILE_COMPAT 2 /* cuFile compatibility mode (POSIX inside cuFile).  Its driver
                                    open hangs without nvidia-fs on this pool's boxes: it runs
                                    under a watchdog (ENDOR_CUFILE_OPEN_TIMEOUT_S, default 10 s)
                                    and a timeout returns ENDOR_ERR_IO instead of hanging;
                                    ENDOR_ALLOW_CUFILE_COMPAT=0 forbids the mode */
#define ENDOR_IO_POSIX 3         /* O_DIRECT reads into two pinned bounce buffers + async H2D */
typedef struct endor_reader endor_reader;
int endor_reader_create(int device_ordinal, size_t bounce_bytes, int mode, endor_reader** out);
int endor_reader_destroy(endor_reader* r);
int endor_reader_mode(const endor_reader* r); /* the ENDOR_IO_* actually in use */
/* Read the bitmap and values sections of `path` (probed into f) into device
 * buffers.  Returns after the data is on the device.  verify != 0 completes
 * decode_endor's checks on the device copy (file_io.hpp:253-270): CRC-32 of
 * the whole file computed on the GPU (BadCrc), padding bits (Malformed),
 * popcount == nnz (CountMismatch); needs a workspace for rows*cols. */
int endor_reader_read(endor_reader* r, const char* path, const endor_file_info* f, void* bitmap_dev,
                      void* values_dev, int verify, void* ws, size_t ws_bytes, void* stream);
/* Cumulative wall time and bytes of endor_reader_read's transfers. */
int endor_reader_stats(const endor_reader* r, double* seconds, uint64_t* bytes);

/* ---- offload pipeline ---------------------------------------------------- */
/* Streams compressed ops from pinned host memory through a double-buffered
 * device staging ring: H2D of op i+1 on the copy stream overlaps decompress
 * + GEMV of op i on the compute stream (the Endor mode stages of
 * sim.hpp:200-204, executed for real and overlapped). */

typedef struct endor_pipeline endor_pipeline;

typedef struct endor_pipeline_op {
    uint64_t rows, cols;
    int32_t dtype;           /* F16; or I8 with flags bit0 (dequantized to f16 on the fly) */
    int32_t flags;           /* bit0: values are i8 quantized with quant_scale (INT8 + Endor,
                                PAPER.md:74): fused dequant + decompress -> f16 W;
                                bit1: materialise W (decompress, then dense GEMV) even when
                                only y is asked for -- by default an f16 op with x/y, no
                                dense_dev and cols % 1024 == 0 runs the fused
                                decompress -> GEMV */
    const void* bitmap_host; /* pinned (cudaHostAlloc / endor_host_alloc) */
    const void* values_host; /* pinned */
    uint64_t nnz;
    const void* x_dev;       /* GEMV input, f16[cols]; NULL = decompress only */
    float* y_dev;            /* GEMV output, f32[rows]; NULL = decompress only */
    void* dense_dev;         /* optional: where the dense W lands (NULL = ring) */
    float* y_host;           /* optional pinned f32[rows]: y is copied back (D2H) */
    float quant_scale;       /* flags bit0 only */
    int32_t reserved2;
    const char* path;        /* non-NULL: the op's bitmap + values come from this .endor file
                                (EndorDirect, SsdToGpu sim.hpp:205-214) through the pipeline's
                                endor_reader instead of bitmap_host / values_host; rows, cols,
                                dtype, nnz must match its header */
    uint64_t tokens;         /* 0 or 1: GEMV as above.  > 1: GEMM (prefill / batched decode):
                                x_dev is f16 [tokens][cols] (cols % 8 == 0), y_dev f32
                                [tokens][rows], y_host (optional) the same size;
                                endor_cuda_gemm_compressed on the compute stream */
    const uint64_t* prefix1024_host; /* optional pinned RankIndex at chunk 1024 (ceil(n/1024)
                                u64, built once at load time like the compression): copied
                                with the op, so the decompress / fused GEMV / GEMM run no
                                counting pass */
    const void* vcode_host;  /* optional coded-values blob in pinned HOST memory (endor_values_encode) of this
                                op's f16 values: crosses the link instead of values_host and is
                                decoded on the compute stream before the decompress / GEMV */
} endor_pipeline_op;

typedef struct endor_pipeline_stats {
    double total_ms;         /* first H2D start -> last op done (device events) */
    double h2d_ms;           /* sum of per-op H2D durations */
    double decompress_ms;    /* sum of per-op decompress durations */
    double gemv_ms;          /* sum of per-op GEMV durations */
    double exposed_compute_ms; /* total_ms minus the copy-engine busy span */
    uint64_t h2d_bytes;
    uint64_t dense_bytes;
    uint64_t kernel_launches;
} endor_pipeline_stats;

/* device_ordinal: CUDA device to use.  max_op_*: largest op the pipeline
 * will see (sizes the ring). */
int endor_pipeline_create(int device_ordinal, uint64_t max_op_elems, int ring_depth,
                          endor_pipeline** out);
int endor_pipeline_destroy(endor_pipeline* p);
/* Run ops[0..nops) in order; asynchronous w.r.t. the host unless sync != 0. */
int endor_pipeline_run(endor_pipeline* p, const endor_pipeline_op* ops, int nops, int sync);
/* Timings of the most recent run (synchronises). */
int endor_pipeline_stats_get(endor_pipeline* p, endor_pipeline_stats* out);
/* The pipeline's compute stream (cudaStream_t as void*). */
void* endor_pipeline_stream(endor_pipeline* p);

/* Pinned host allocation helpers (cudaHostAlloc, portable). */
void* endor_host_alloc(size_t bytes);
void endor_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* ENDOR_CUDA_H */
