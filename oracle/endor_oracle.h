/*
 * endor_oracle.h -- CPU restatement of the reference's bitmap-sparse codec.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it, and only as the checker.  The product
 * path (paper_2406_11674_b200/) never links or calls it.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/include/endor/).
 * Parity of this restatement is pinned by tests/test_oracle.py against the
 * golden vectors in tests/golden/ (produced by the reference itself via
 * oracle/_ref/libendor_ref.so, see tests/golden/make_golden.py) and against
 * the reference's own literal KATs (test_codec.cpp, test_bitmap.cpp,
 * test_weight_gen.cpp).
 */
#ifndef ENDOR_ORACLE_H
#define ENDOR_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror include/endor_cuda.h (and the reference's exception
 * classes, error.hpp:9-63). */
enum {
    OR_OK = 0,
    OR_SIZE = 1,        /* SizeError        error.hpp:15 */
    OR_CORRUPTION = 2,  /* CorruptionError  error.hpp:22 */
    OR_BOUNDS = 3,      /* BoundsError      error.hpp:28 */
    OR_INVALID = 4,     /* std::invalid_argument */
};

/* Bitmap::count (bitmap.hpp:34-38): popcount of the first n bits. */
uint64_t or_popcount(const uint8_t* bitmap, uint64_t n);

/* Bitmap::rank_range (bitmap.hpp:44-61). */
uint64_t or_rank_range(const uint8_t* bitmap, uint64_t begin, uint64_t end);

/* build_rank_index (bitmap.hpp:117-132).  prefix_out holds ceil(n/cs)
 * entries.  Returns OR_INVALID for a chunk size that is not a power of two
 * >= 64 (bitmap.hpp:118-120). */
int or_rank_index(const uint8_t* bitmap, uint64_t n, uint64_t chunk_size, uint64_t* prefix_out);

/* decompress (codec.hpp:157-166) = popcount check + scatter_range over
 * [0, n) (codec.hpp:132-152).  dst holds n*eb bytes. */
int or_decompress(uint64_t rows, uint64_t cols, int eb, const uint8_t* bitmap,
                  const uint8_t* values, uint64_t nnz, uint8_t* dst);

/* detail::scatter_range (codec.hpp:132-152). */
void or_scatter_range(int eb, const uint8_t* bitmap, const uint8_t* values, uint64_t begin,
                      uint64_t end, uint64_t value_offset, uint8_t* dst);

/* detail::check_index (codec.hpp:170-184). */
int or_check_index(uint64_t n, const uint8_t* bitmap, uint64_t nnz, uint64_t chunk_size,
                   const uint64_t* prefix, uint64_t chunk_count);

/* decompress_chunk_into (codec.hpp:191-201). */
int or_decompress_chunk_into(uint64_t rows, uint64_t cols, int eb, const uint8_t* bitmap,
                             const uint8_t* values, uint64_t nnz, uint64_t chunk_size,
                             const uint64_t* prefix, uint64_t chunk_count, uint64_t k,
                             uint8_t* dst, uint64_t dst_bytes);

/* decompress_chunked (codec.hpp:205-216). */
int or_decompress_chunked(uint64_t rows, uint64_t cols, int eb, const uint8_t* bitmap,
                          const uint8_t* values, uint64_t nnz, uint64_t chunk_size,
                          const uint64_t* prefix, uint64_t chunk_count, uint8_t* dst);

/* compress (codec.hpp:97-126).  bitmap_out: ceil(n/8) bytes (zeroed here);
 * values_out: capacity n*eb.  Writes nnz and the negative-zero flag. */
int or_compress(uint64_t rows, uint64_t cols, int eb, const uint8_t* dense, uint8_t* bitmap_out,
                uint8_t* values_out, uint64_t* nnz_out, int* negzero_out);

/* f16 bit math (float16.hpp:12-73). */
float or_f16_to_f32(uint16_t h);
uint16_t or_f32_to_f16(float f);

/* synth_weight (weight_gen.hpp:40-55) with SplitMix64 (weight_gen.hpp:17-36). */
void or_synth_weight(uint64_t n, int eb, uint64_t seed, uint8_t* out);

/* magnitude_prune (weight_gen.hpp:96-113, impl 78-89).  Restated as an exact
 * threshold selection: the reference's nth_element picks the floor(s*n)
 * smallest elements under the total order (key, index); that set is unique,
 * so a histogram threshold + in-order tie cut selects the identical set. */
int or_magnitude_prune(uint64_t n, int eb, double sparsity, const uint8_t* in, uint8_t* out);

/* nm_prune (weight_gen.hpp:118-141). */
int or_nm_prune(uint64_t rows, uint64_t cols, int eb, uint64_t nkeep, uint64_t m,
                const uint8_t* in, uint8_t* out);

/* std::mt19937_64 + libstdc++ generate_canonical<double,53>, as used by the
 * reference's test generators (test_helpers.hpp:15-38, acceptance.cpp:53-74). */
typedef struct { uint64_t mt[312]; int idx; } or_mt64;
void or_mt64_seed(or_mt64* g, uint64_t seed);
uint64_t or_mt64_next(or_mt64* g);
double or_mt64_coin(or_mt64* g);

/* endor::test::random_dense (test_helpers.hpp:15-38). */
void or_random_dense(uint64_t rows, uint64_t cols, int eb, uint64_t seed, double zero_fraction,
                     uint8_t* out);

/* acceptance.cpp:53-74 random_matrix (consumes the caller's generator). */
void or_acceptance_matrix(or_mt64* g, uint64_t rows, uint64_t cols, int eb, double zero_fraction,
                          uint8_t* out);

/* dequantize_values (codec.hpp:334-349): i8 * scale -> f16 (RNE). */
void or_dequantize_values(const uint8_t* q, uint64_t nnz, float scale, uint16_t* out);

/* quantize_values (codec.hpp:306-331): symmetric absmax f16 -> i8; returns
 * the scale (1.0 for an all-zero tensor). */
float or_quantize_values(const uint16_t* vals, uint64_t nnz, uint8_t* q_out);

/* Multi-threaded decompress_chunk_into fan-out (the reference's documented
 * parallel contract, codec.hpp:188-190/203-204) used as the "port" CPU
 * baseline when oracle/_ref is unavailable.  Returns seconds. */
double or_decompress_parallel(uint64_t n, int eb, const uint8_t* bitmap, const uint8_t* values,
                              uint64_t chunk_size, const uint64_t* prefix, uint8_t* dst,
                              int threads);

/* synth_weight -> magnitude_prune -> compress for one f16 op, multi-threaded
 * (identical output to the single-threaded functions above; used to build
 * the --impl reference arm's inputs on the CPU).  bitmap_out: ceil(n/8)
 * bytes; values_out: capacity n*2.  Returns nnz. */
uint64_t or_make_op_mt(uint64_t rows, uint64_t cols, uint64_t seed, double sparsity, int threads,
                       uint8_t* bitmap_out, uint8_t* values_out);

/* fp32 GEMV reference y = W x over f16 W [rows, cols] row-major (the
 * consumer the reference only models as a constant, sim.hpp:227). */
void or_gemv_f16(uint64_t rows, uint64_t cols, const uint16_t* w, const uint16_t* x, float* y);

#ifdef __cplusplus
}
#endif
#endif
