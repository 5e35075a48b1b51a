// ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile directly against
// /root/reference/proj/include (never copied) into oracle/_ref/libendor_ref.so.
// It exists so the oracle restatement (endor_oracle.c) can be validated
// against the reference itself, golden vectors can be generated
// (tests/golden/make_golden.py), and bench.py can time the reference's own
// CPU decompress as its cpu_baseline / --impl reference arm.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "endor/endor.hpp"
#include "test_helpers.hpp"

using namespace endor;

namespace {

Dtype dt(int eb) { return eb == 2 ? Dtype::F16 : Dtype::I8; }

int code_of(const std::exception& e) {
    if (dynamic_cast<const SizeError*>(&e)) return 1;
    if (dynamic_cast<const CorruptionError*>(&e)) return 2;
    if (dynamic_cast<const BoundsError*>(&e)) return 3;
    if (dynamic_cast<const std::invalid_argument*>(&e)) return 4;
    if (dynamic_cast<const FormatError*>(&e)) return 10 + static_cast<int>(dynamic_cast<const FormatError*>(&e)->kind());
    return 9;
}

EndorTensor make_tensor(uint64_t rows, uint64_t cols, int eb, const uint8_t* bitmap,
                        const uint8_t* values, uint64_t nnz) {
    const uint64_t n = checked_element_count(rows, cols);
    auto bb = std::span<const std::byte>(reinterpret_cast<const std::byte*>(bitmap), (n + 7) / 8);
    Bitmap b = Bitmap::from_bytes(bb, n);
    std::vector<std::byte> v(reinterpret_cast<const std::byte*>(values),
                             reinterpret_cast<const std::byte*>(values) + nnz * eb);
    return EndorTensor(rows, cols, dt(eb), std::move(b), std::move(v));
}

}  // namespace

extern "C" {

// Opaque tensor handle so timing excludes construction.
void* ref_tensor_new(uint64_t rows, uint64_t cols, int eb, const uint8_t* bitmap,
                     const uint8_t* values, uint64_t nnz, int* status) {
    try {
        *status = 0;
        return new EndorTensor(make_tensor(rows, cols, eb, bitmap, values, nnz));
    } catch (const std::exception& e) {
        *status = code_of(e);
        return nullptr;
    }
}

void ref_tensor_free(void* t) { delete static_cast<EndorTensor*>(t); }

// endor::decompress (codec.hpp:157) as shipped: 1 thread, includes the
// DenseMatrix allocation.  Returns the wall seconds of the call; copies the
// result into dst when dst != nullptr (outside the timed region).
double ref_decompress_timed(void* th, uint8_t* dst, int* status) {
    try {
        const EndorTensor& t = *static_cast<EndorTensor*>(th);
        auto t0 = std::chrono::steady_clock::now();
        DenseMatrix out = decompress(t);
        auto t1 = std::chrono::steady_clock::now();
        if (dst && out.size_bytes()) std::memcpy(dst, out.bytes().data(), out.size_bytes());
        *status = 0;
        return std::chrono::duration<double>(t1 - t0).count();
    } catch (const std::exception& e) {
        *status = code_of(e);
        return -1.0;
    }
}

// The reference's documented parallel contract (codec.hpp:188-190,203-204):
// decompress_chunk_into over all chunks fanned across `threads` std::threads
// into a caller-owned, pre-faulted buffer.  Returns wall seconds.
double ref_decompress_parallel_timed(void* th, const uint64_t* prefix, uint64_t chunk_size,
                                     uint64_t chunk_count, int threads, uint8_t* dst,
                                     int* status) {
    try {
        const EndorTensor& t = *static_cast<EndorTensor*>(th);
        RankIndex idx(chunk_size, std::vector<uint64_t>(prefix, prefix + chunk_count));
        std::span<std::byte> span(reinterpret_cast<std::byte*>(dst), t.dense_bytes());
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int w = 0; w < threads; ++w) {
            pool.emplace_back([&, w] {
                const uint64_t k0 = chunk_count * w / threads, k1 = chunk_count * (w + 1) / threads;
                for (uint64_t k = k0; k < k1; ++k) decompress_chunk_into(t, idx, k, span);
            });
        }
        for (auto& p : pool) p.join();
        auto t1 = std::chrono::steady_clock::now();
        *status = 0;
        return std::chrono::duration<double>(t1 - t0).count();
    } catch (const std::exception& e) {
        *status = code_of(e);
        return -1.0;
    }
}

int ref_decompress(uint64_t rows, uint64_t cols, int eb, const uint8_t* bitmap,
                   const uint8_t* values, uint64_t nnz, uint8_t* dst) {
    try {
        DenseMatrix out = decompress(make_tensor(rows, cols, eb, bitmap, values, nnz));
        if (out.size_bytes()) std::memcpy(dst, out.bytes().data(), out.size_bytes());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_rank_index(const uint8_t* bitmap, uint64_t n, uint64_t chunk_size, uint64_t* prefix) {
    try {
        Bitmap b = Bitmap::from_bytes(
            std::span<const std::byte>(reinterpret_cast<const std::byte*>(bitmap), (n + 7) / 8), n);
        RankIndex idx = build_rank_index(b, chunk_size);
        std::copy(idx.prefix().begin(), idx.prefix().end(), prefix);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_decompress_chunked(uint64_t rows, uint64_t cols, int eb, const uint8_t* bitmap,
                           const uint8_t* values, uint64_t nnz, uint64_t chunk_size,
                           const uint64_t* prefix, uint64_t chunk_count, uint8_t* dst) {
    try {
        EndorTensor t = make_tensor(rows, cols, eb, bitmap, values, nnz);
        RankIndex idx(chunk_size, std::vector<uint64_t>(prefix, prefix + chunk_count));
        DenseMatrix out = decompress_chunked(t, idx);
        if (out.size_bytes()) std::memcpy(dst, out.bytes().data(), out.size_bytes());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_decompress_chunk_into(uint64_t rows, uint64_t cols, int eb, const uint8_t* bitmap,
                              const uint8_t* values, uint64_t nnz, uint64_t chunk_size,
                              const uint64_t* prefix, uint64_t chunk_count, uint64_t k,
                              uint8_t* dst, uint64_t dst_bytes) {
    try {
        EndorTensor t = make_tensor(rows, cols, eb, bitmap, values, nnz);
        RankIndex idx(chunk_size, std::vector<uint64_t>(prefix, prefix + chunk_count));
        decompress_chunk_into(t, idx, k,
                              std::span<std::byte>(reinterpret_cast<std::byte*>(dst), dst_bytes));
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// compress (codec.hpp:97): values_out needs n*eb capacity.
int ref_compress(uint64_t rows, uint64_t cols, int eb, const uint8_t* dense, uint8_t* bitmap_out,
                 uint8_t* values_out, uint64_t* nnz, int* negzero) {
    try {
        std::vector<std::byte> d(reinterpret_cast<const std::byte*>(dense),
                                 reinterpret_cast<const std::byte*>(dense) + rows * cols * eb);
        EndorTensor t = compress(DenseMatrix(rows, cols, dt(eb), std::move(d)));
        auto bm = t.bitmap().to_bytes();
        if (!bm.empty()) std::memcpy(bitmap_out, bm.data(), bm.size());
        if (t.values_bytes()) std::memcpy(values_out, t.values().data(), t.values_bytes());
        *nnz = t.nnz();
        *negzero = t.negative_zero_collapsed();
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// synth_weight (weight_gen.hpp:40) + optional magnitude_prune (:96).
int ref_synth_prune(uint64_t rows, uint64_t cols, int eb, uint64_t seed, double sparsity,
                    uint8_t* out) {
    try {
        OpShape s{"op", rows, cols, dt(eb)};
        DenseMatrix w = synth_weight(s, seed);
        if (sparsity > 0.0) w = magnitude_prune(w, sparsity);
        if (w.size_bytes()) std::memcpy(out, w.bytes().data(), w.size_bytes());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_nm_prune(uint64_t rows, uint64_t cols, int eb, const uint8_t* in, uint64_t n, uint64_t m,
                 uint8_t* out) {
    try {
        std::vector<std::byte> d(reinterpret_cast<const std::byte*>(in),
                                 reinterpret_cast<const std::byte*>(in) + rows * cols * eb);
        DenseMatrix w = nm_prune(DenseMatrix(rows, cols, dt(eb), std::move(d)), n, m);
        if (w.size_bytes()) std::memcpy(out, w.bytes().data(), w.size_bytes());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// endor::test::random_dense (tests/test_helpers.hpp:15-38), included from the
// reference's own test tree; used to cross-check the oracle's
// mt19937_64/generate_canonical port.
int ref_random_dense(uint64_t rows, uint64_t cols, int eb, uint64_t seed, double zf,
                     uint8_t* out) {
    DenseMatrix w = endor::test::random_dense(rows, cols, dt(eb), seed, zf);
    if (w.size_bytes()) std::memcpy(out, w.bytes().data(), w.size_bytes());
    return 0;
}

uint64_t ref_mt64_draws(uint64_t seed, uint64_t count, uint64_t* out, double* coins) {
    std::mt19937_64 a(seed), b(seed);
    std::uniform_real_distribution<double> coin(0.0, 1.0);
    for (uint64_t i = 0; i < count; ++i) {
        out[i] = a();
        coins[i] = coin(b);
    }
    return count;
}

// .endor container (file_io.hpp:187-277).
uint64_t ref_encode_endor(uint64_t rows, uint64_t cols, int eb, const uint8_t* bitmap,
                          const uint8_t* values, uint64_t nnz, int negzero, uint8_t* out,
                          uint64_t cap) {
    EndorTensor t0 = make_tensor(rows, cols, eb, bitmap, values, nnz);
    EndorTensor t(rows, cols, dt(eb), t0.bitmap(),
                  std::vector<std::byte>(t0.values().begin(), t0.values().end()), std::nullopt,
                  negzero != 0);
    auto data = encode_endor(t);
    if (data.size() <= cap) std::memcpy(out, data.data(), data.size());
    return data.size();
}

// Returns 0 on success, 10+Kind for FormatError; fills header fields.
int ref_decode_endor(const uint8_t* data, uint64_t size, uint64_t* rows, uint64_t* cols,
                     int* eb, uint64_t* nnz) {
    try {
        EndorTensor t = decode_endor(
            std::span<const std::byte>(reinterpret_cast<const std::byte*>(data), size));
        *rows = t.rows();
        *cols = t.cols();
        *eb = static_cast<int>(elem_bytes(t.dtype()));
        *nnz = t.nnz();
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

uint16_t ref_f32_to_f16(float f) { return f32_to_f16(f); }

// extract_rows / extract_cols (codec.hpp:239-297); returns the error code.
int ref_extract(uint64_t rows, uint64_t cols, int eb, const uint8_t* bitmap, const uint8_t* values, uint64_t nnz,
                const uint64_t* sel, uint64_t nsel, int by_rows, uint8_t* out) {
    try {
        EndorTensor t = make_tensor(rows, cols, eb, bitmap, values, nnz);
        std::vector<std::size_t> s(sel, sel + nsel);
        DenseMatrix m = by_rows ? extract_rows(t, s) : extract_cols(t, s);
        if (m.size_bytes()) std::memcpy(out, m.bytes().data(), m.size_bytes());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// quantize_values (codec.hpp:306-331) of an f16 tensor: writes the i8 values,
// returns the scale.
float ref_quantize_values(uint64_t rows, uint64_t cols, const uint8_t* bitmap, const uint8_t* values,
                          uint64_t nnz, uint8_t* q_out) {
    EndorTensor q = quantize_values(make_tensor(rows, cols, 2, bitmap, values, nnz));
    if (q.values_bytes()) std::memcpy(q_out, q.values().data(), q.values_bytes());
    return *q.quant_scale();
}

// decompress(dequantize_values(t)) (codec.hpp:334-349 then :157) for an i8
// tensor with a quantization scale; dst receives n f16 values.
int ref_decompress_dequant(uint64_t rows, uint64_t cols, const uint8_t* bitmap, const uint8_t* q,
                           uint64_t nnz, float scale, uint8_t* dst) {
    try {
        EndorTensor t0 = make_tensor(rows, cols, 1, bitmap, q, nnz);
        EndorTensor t(rows, cols, Dtype::I8, t0.bitmap(),
                      std::vector<std::byte>(t0.values().begin(), t0.values().end()), scale);
        DenseMatrix out = decompress(dequantize_values(t));
        if (out.size_bytes()) std::memcpy(dst, out.bytes().data(), out.size_bytes());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

}  // extern "C"
