// endor_cuda.hpp -- the reference's own C++ codec signatures, executed on a
// B200 through the C ABI (endor_cuda.h).
//
// Drop-in for reference code that includes "endor/endor.hpp": replace
//     endor::decompress(t)                 (codec.hpp:157)
//     endor::decompress_chunked(t, idx)    (codec.hpp:205)
//     endor::decompress_chunk_into(...)    (codec.hpp:191)
//     endor::build_rank_index(b, cs)       (bitmap.hpp:117)
//     endor::compress(w)                   (codec.hpp:97)
//     endor::extract_rows(t, rows)         (codec.hpp:239)
//     endor::extract_cols(t, cols)         (codec.hpp:271)
//     endor::quantize_values(t)            (codec.hpp:306)
//     endor::dequantize_values(t)          (codec.hpp:334)
// with the same calls in namespace endor::cuda.  Arguments, return types,
// ownership (value semantics, caller-owned span for chunk_into) and the
// exception types thrown (error.hpp) are the reference's.  Requires the
// reference's headers on the include path and links libendor_cuda.so; no
// CUDA headers are needed by the caller.
#pragma once

#include <bit>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "endor/codec.hpp"
#include "endor_cuda.h"

namespace endor::cuda {

// Map an endor_status onto the reference's exception classes (error.hpp:9-63).
inline void check(int status) {
    if (status == ENDOR_OK) return;
    const std::string what = endor_cuda_last_error_string();
    switch (status) {
        case ENDOR_ERR_SIZE: throw SizeError(what);
        case ENDOR_ERR_CORRUPTION: throw CorruptionError(what);
        case ENDOR_ERR_BOUNDS: throw BoundsError(what);
        case ENDOR_ERR_INVALID_ARGUMENT: throw std::invalid_argument(what);
        case ENDOR_ERR_CONFIG: throw ConfigError(what);
        default: throw Error("CUDA: " + what);
    }
}

inline int32_t dtype_code(Dtype d) { return static_cast<int32_t>(d); }

// The bitmap's serialized bytes (bitmap.hpp:65-70: ceil(size/8) bytes,
// LSB-first) without a copy: Bitmap stores them as little-endian u64 words.
inline const std::byte* bitmap_bytes(const Bitmap& b) {
    static_assert(std::endian::native == std::endian::little, "Bitmap words are read as LSB-first bytes");
    return reinterpret_cast<const std::byte*>(b.words().data());
}

// decompress (codec.hpp:157-166).  The reference re-checks values vs popcount
// first (:158-160); EndorTensor's constructor already guarantees it and the
// device re-verifies popcount == nnz.
inline DenseMatrix decompress(const EndorTensor& t) {
    if (t.values_bytes() != t.nnz() * elem_bytes(t.dtype()))
        throw CorruptionError("values length does not match bitmap popcount");
    DenseMatrix out(t.rows(), t.cols(), t.dtype());
    if (t.element_count() == 0) return out;
    const std::byte* bm = bitmap_bytes(t.bitmap());
    check(endor_cuda_decompress_host(t.rows(), t.cols(), dtype_code(t.dtype()), bm,
                                     t.values().data(), t.nnz(), out.bytes().data()));
    return out;
}

// build_rank_index (bitmap.hpp:117-132).
inline RankIndex build_rank_index(const Bitmap& bitmap, std::uint64_t chunk_size) {
    if (chunk_size < 64 || (chunk_size & (chunk_size - 1)) != 0)
        throw std::invalid_argument("chunk_size must be a power of two >= 64");
    const std::uint64_t n = bitmap.size();
    const std::uint64_t chunks = n == 0 ? 0 : (n + chunk_size - 1) / chunk_size;
    std::vector<std::uint64_t> prefix(chunks);
    if (chunks) {
        check(endor_cuda_rank_index_host(bitmap_bytes(bitmap), n, chunk_size, prefix.data()));
    }
    return RankIndex(chunk_size, std::move(prefix));
}

// decompress_chunked (codec.hpp:205-216).
inline DenseMatrix decompress_chunked(const EndorTensor& t, const RankIndex& idx) {
    DenseMatrix out(t.rows(), t.cols(), t.dtype());
    const std::byte* bm = bitmap_bytes(t.bitmap());
    check(endor_cuda_decompress_chunked_host(t.rows(), t.cols(), dtype_code(t.dtype()), bm,
                                             t.values().data(), t.nnz(), idx.chunk_size(),
                                             idx.prefix().data(), idx.chunk_count(),
                                             out.bytes().data()));
    return out;
}

// decompress_chunk_into (codec.hpp:191-201): writes exactly chunk k's range.
inline void decompress_chunk_into(const EndorTensor& t, const RankIndex& idx, std::uint64_t k,
                                  std::span<std::byte> dst) {
    const std::byte* bm = bitmap_bytes(t.bitmap());
    check(endor_cuda_decompress_chunk_into_host(t.rows(), t.cols(), dtype_code(t.dtype()), bm,
                                                t.values().data(), t.nnz(), idx.chunk_size(),
                                                idx.prefix().data(), idx.chunk_count(), k, dst.data(),
                                                dst.size()));
}

// compress (codec.hpp:97-126).
inline EndorTensor compress(const DenseMatrix& w) {
    const std::uint64_t n = checked_element_count(w.rows(), w.cols());
    std::vector<std::byte> bm((n + 7) / 8);
    std::vector<std::byte> vals(w.size_bytes());
    std::uint64_t nnz = 0;
    int32_t negzero = 0;
    check(endor_cuda_compress_host(w.rows(), w.cols(), dtype_code(w.dtype()), w.bytes().data(),
                                   bm.data(), vals.data(), &nnz, &negzero));
    vals.resize(nnz * elem_bytes(w.dtype()));
    return EndorTensor(w.rows(), w.cols(), w.dtype(), Bitmap::from_bytes(bm, n), std::move(vals),
                       std::nullopt, negzero != 0);
}

// extract_rows / extract_cols (codec.hpp:239-297): index checks in the
// reference's order and exception types (check_sorted_unique, :224-232).
inline DenseMatrix extract_rows(const EndorTensor& t, std::span<const std::size_t> rows) {
    DenseMatrix out(rows.size(), t.cols(), t.dtype());
    const std::byte* bm = bitmap_bytes(t.bitmap());
    const std::vector<std::uint64_t> sel(rows.begin(), rows.end());
    check(endor_cuda_extract_rows_host(t.rows(), t.cols(), dtype_code(t.dtype()), bm, t.values().data(),
                                       t.nnz(), sel.data(), sel.size(), out.bytes().data()));
    return out;
}

inline DenseMatrix extract_cols(const EndorTensor& t, std::span<const std::size_t> cols) {
    DenseMatrix out(t.rows(), cols.size(), t.dtype());
    const std::byte* bm = bitmap_bytes(t.bitmap());
    const std::vector<std::uint64_t> sel(cols.begin(), cols.end());
    check(endor_cuda_extract_cols_host(t.rows(), t.cols(), dtype_code(t.dtype()), bm, t.values().data(),
                                       t.nnz(), sel.data(), sel.size(), out.bytes().data()));
    return out;
}

// quantize_values (codec.hpp:306-331): symmetric absmax f16 -> i8 of the
// packed values; the bitmap is shared.
inline EndorTensor quantize_values(const EndorTensor& t) {
    if (t.dtype() != Dtype::F16) throw std::invalid_argument("quantize_values requires an f16 tensor");
    std::vector<std::byte> q(t.nnz());
    float scale = 1.0f;
    check(endor_cuda_quantize_values_host(t.values().data(), t.nnz(), q.data(), &scale));
    return EndorTensor(t.rows(), t.cols(), Dtype::I8, t.bitmap(), std::move(q), scale,
                       t.negative_zero_collapsed());
}

// dequantize_values (codec.hpp:334-349).  decompress(dequantize_values(t)) is
// also available fused on device (endor_cuda_decompress_dequant).
inline EndorTensor dequantize_values(const EndorTensor& t) {
    if (t.dtype() != Dtype::I8 || !t.quant_scale())
        throw std::invalid_argument("dequantize_values requires a quantized i8 tensor");
    std::vector<std::byte> out(t.nnz() * 2);
    check(endor_cuda_dequantize_values_host(t.values().data(), t.nnz(), *t.quant_scale(), out.data()));
    return EndorTensor(t.rows(), t.cols(), Dtype::F16, t.bitmap(), std::move(out), std::nullopt,
                       t.negative_zero_collapsed());
}

}  // namespace endor::cuda
