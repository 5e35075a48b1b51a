// ref_parity.cpp -- reference-style C++ parity suite for the drop-in boundary.
//
// TEST INFRASTRUCTURE.  Built by oracle/Makefile into oracle/_ref/ref_parity
// against the UNMODIFIED reference headers (oracle side) and
// include/endor_cuda.hpp (CUDA side, linking libendor_cuda.so); run on a GPU
// box by tests/test_gpu_cpp_parity.py.  Each case restates an assertion of
// the reference's test_codec.cpp / test_bitmap.cpp / acceptance.cpp with
// endor::X replaced by endor::cuda::X and the reference's own result as the
// oracle.  Prints one PASS/FAIL line per case; exit code = failures.
#include <cstdio>
#include <functional>
#include <random>
#include <string>

#include "endor/endor.hpp"
#include "endor_cuda.hpp"
#include "test_helpers.hpp"

using namespace endor;
using endor::test::random_dense;

static int g_fail = 0;

#define REQUIRE(cond)                                                              \
    do {                                                                           \
        if (!(cond)) throw std::runtime_error(std::string("REQUIRE failed: ") + #cond); \
    } while (0)

template <class E, class F>
static bool throws_as(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static void run(const char* name, const std::function<void()>& body) {
    try {
        body();
        std::printf("[PASS] %s\n", name);
    } catch (const std::exception& e) {
        ++g_fail;
        std::printf("[FAIL] %s -- %s\n", name, e.what());
    }
    std::fflush(stdout);
}

int main() {
    run("hand-built 2x2 bitmap 1010 (test_codec.cpp:138-145)", [] {
        Bitmap b(4);
        b.set(0);
        b.set(2);
        std::vector<std::byte> v(4);
        const uint16_t v0 = 0x3C00, v1 = 0x4200;
        std::memcpy(v.data(), &v0, 2);
        std::memcpy(v.data() + 2, &v1, 2);
        const EndorTensor t(2, 2, Dtype::F16, b, v);
        const DenseMatrix out = cuda::decompress(t);
        REQUIRE(out.get_u16(0) == 0x3C00 && out.get_u16(1) == 0 && out.get_u16(2) == 0x4200 &&
                out.get_u16(3) == 0);
        REQUIRE(out == decompress(t));
    });
    run("empty tensor decompresses to zeros (test_codec.cpp:132-136)", [] {
        const EndorTensor t(3, 3, Dtype::F16, Bitmap(9), {});
        REQUIRE(cuda::decompress(t) == decompress(t));
    });
    run("NaN payload / -inf survive (test_codec.cpp:123-130)", [] {
        DenseMatrix w(1, 3, Dtype::F16);
        w.set_u16(0, 0x7E01);
        w.set_u16(2, 0xFC00);
        REQUIRE(cuda::decompress(compress(w)) == w);
        REQUIRE(cuda::decompress(cuda::compress(w)) == w);
    });
    run("negative zero pruned and flagged (test_codec.cpp:110-121)", [] {
        DenseMatrix w(2, 2, Dtype::F16);
        w.set_u16(0, 0x8000);
        w.set_u16(1, 0xBC00);
        const EndorTensor t = cuda::compress(w);
        REQUIRE(t.negative_zero_collapsed() && t.nnz() == 1);
        REQUIRE(cuda::decompress(t) == canonicalize_zeros(w));
    });
    run("round trips across shapes/sparsities/dtypes (test_codec.cpp:51-62)", [] {
        std::mt19937_64 rng(7);
        for (int iter = 0; iter < 60; ++iter) {
            const std::size_t rows = 1 + rng() % 33, cols = 1 + rng() % 33;
            const Dtype dt = rng() % 2 ? Dtype::F16 : Dtype::I8;
            const double zeros = static_cast<double>(rng() % 101) / 100.0;
            const DenseMatrix w = random_dense(rows, cols, dt, rng(), zeros);
            const EndorTensor tr = compress(w);
            const EndorTensor tc = cuda::compress(w);
            REQUIRE(tc.bitmap() == tr.bitmap());
            REQUIRE(std::equal(tc.values().begin(), tc.values().end(), tr.values().begin(), tr.values().end()));
            REQUIRE(cuda::decompress(tr) == w);
        }
    });
    run("chunked == scalar at 64/256/4096/8192 (test_codec.cpp:155-166)", [] {
        const DenseMatrix w = random_dense(37, 200, Dtype::F16, 3, 0.6);
        const EndorTensor t = compress(w);
        for (std::uint64_t cs : {64ull, 256ull, 4096ull, 8192ull}) {
            const RankIndex ri = build_rank_index(t.bitmap(), cs);
            const RankIndex ci = cuda::build_rank_index(t.bitmap(), cs);
            REQUIRE(ri.prefix() == ci.prefix());
            REQUIRE(cuda::decompress_chunked(t, ci) == w);
        }
    });
    run("chunks in any order (test_codec.cpp:168-179)", [] {
        const DenseMatrix w = random_dense(16, 100, Dtype::I8, 21, 0.5);
        const EndorTensor t = compress(w);
        const RankIndex idx = build_rank_index(t.bitmap(), 128);
        std::vector<std::byte> buf(t.dense_bytes());
        for (std::size_t k = idx.chunk_count(); k-- > 0;) cuda::decompress_chunk_into(t, idx, k, buf);
        REQUIRE(buf == std::vector<std::byte>(w.bytes().begin(), w.bytes().end()));
    });
    run("a chunk writes exactly its own region (test_codec.cpp:181-200)", [] {
        const DenseMatrix w = random_dense(8, 64, Dtype::F16, 5, 0.4);
        const EndorTensor t = compress(w);
        const RankIndex idx = build_rank_index(t.bitmap(), 128);
        for (std::size_t k = 0; k < idx.chunk_count(); ++k) {
            std::vector<std::byte> a(t.dense_bytes(), std::byte{0xAB}), b(a);
            decompress_chunk_into(t, idx, k, a);
            cuda::decompress_chunk_into(t, idx, k, b);
            REQUIRE(a == b);
        }
    });
    run("mismatched / truncated index rejected (test_codec.cpp:202-213)", [] {
        const DenseMatrix w = random_dense(10, 10, Dtype::F16, 9, 0.5);
        const EndorTensor t = compress(w);
        const RankIndex bad = build_rank_index(compress(random_dense(10, 10, Dtype::F16, 10, 0.2)).bitmap(), 64);
        REQUIRE(throws_as<CorruptionError>([&] { cuda::decompress_chunked(t, bad); }));
        const RankIndex ok = build_rank_index(t.bitmap(), 64);
        RankIndex trunc(64, std::vector<std::uint64_t>(ok.prefix().begin(), ok.prefix().end() - 1));
        REQUIRE(throws_as<CorruptionError>([&] { cuda::decompress_chunked(t, trunc); }));
        std::vector<std::byte> buf(t.dense_bytes());
        REQUIRE(throws_as<BoundsError>([&] { cuda::decompress_chunk_into(t, ok, ok.chunk_count(), buf); }));
        std::vector<std::byte> small(t.dense_bytes() - 2);
        REQUIRE(throws_as<std::invalid_argument>([&] { cuda::decompress_chunk_into(t, ok, 0, small); }));
        REQUIRE(throws_as<CorruptionError>([&] { cuda::decompress_chunk_into(t, bad, 99, buf); }));
    });
    run("rank index KATs + chunk-size validation (test_bitmap.cpp:77-105)", [] {
        Bitmap b(256);
        for (std::uint64_t i = 0; i < 256; i += 2) b.set(i);
        REQUIRE(cuda::build_rank_index(b, 64).prefix() == (std::vector<std::uint64_t>{0, 32, 64, 96}));
        REQUIRE(cuda::build_rank_index(Bitmap(300), 128).prefix() == (std::vector<std::uint64_t>{0, 0, 0}));
        for (std::uint64_t cs : {32ull, 96ull, 0ull})
            REQUIRE(throws_as<std::invalid_argument>([&] { cuda::build_rank_index(Bitmap(128), cs); }));
    });
    run("acceptance criterion 3 generator, 300 cases (acceptance.cpp:99-125)", [] {
        std::mt19937_64 rng(20240521);
        std::uniform_real_distribution<double> coin(0.0, 1.0);
        for (int iter = 0; iter < 300; ++iter) {
            const std::size_t rows = 1 + rng() % (iter % 50 == 0 ? 160 : 48);
            const std::size_t cols = 1 + rng() % (iter % 50 == 0 ? 160 : 48);
            const Dtype dt = rng() % 2 ? Dtype::F16 : Dtype::I8;
            const double zeros = static_cast<double>(rng() % 101) / 100.0;
            DenseMatrix w(rows, cols, dt);
            for (std::size_t i = 0; i < w.element_count(); ++i) {
                if (coin(rng) < zeros) continue;
                if (dt == Dtype::F16) {
                    std::uint16_t v;
                    do { v = static_cast<std::uint16_t>(rng()); } while ((v & 0x7FFFu) == 0);
                    w.set_u16(i, v);
                } else {
                    std::int8_t v;
                    do { v = static_cast<std::int8_t>(rng()); } while (v == 0);
                    w.set_i8(i, v);
                }
            }
            const EndorTensor t = compress(w);
            REQUIRE(cuda::decompress(t) == decompress(t));
            const std::uint64_t chunk = 64ull << (rng() % 7);
            const RankIndex idx = cuda::build_rank_index(t.bitmap(), chunk);
            REQUIRE(idx.prefix() == build_rank_index(t.bitmap(), chunk).prefix());
            REQUIRE(cuda::decompress_chunked(t, idx) == decompress_chunked(t, idx));
            for (std::size_t r = 0; r < rows; ++r) (void)coin(rng);
            for (std::size_t c = 0; c < cols; ++c) (void)coin(rng);
        }
    });
    run("fc1-shaped tensor 9216x36864 @50% (acceptance.cpp:77-92 sizes)", [] {
        const OpShape s{"fc1", 9216, 36864, Dtype::F16};
        const DenseMatrix w = synth_weight(s, 7);
        // pruned on the GPU bit-exactly, then compressed by the REFERENCE
        DenseMatrix p = magnitude_prune(w, 0.5);
        const EndorTensor t = compress(p);
        REQUIRE(t.values_bytes() == 339738624ull && t.bitmap_bytes() == 42467328ull);
        REQUIRE(cuda::decompress(t) == p);
    });
    run("extract_rows / extract_cols == slices of decompress (acceptance.cpp:126-153)", [] {
        std::mt19937_64 rng(99);
        for (int iter = 0; iter < 40; ++iter) {
            const std::size_t rows = 1 + rng() % 40, cols = 1 + rng() % 3000;
            const Dtype dt = rng() % 2 ? Dtype::F16 : Dtype::I8;
            const DenseMatrix w = random_dense(rows, cols, dt, rng(), static_cast<double>(rng() % 101) / 100.0);
            const EndorTensor t = compress(w);
            std::vector<std::size_t> rs, cs;
            for (std::size_t r = 0; r < rows; ++r) if (rng() % 3 == 0) rs.push_back(r);
            for (std::size_t c = 0; c < cols; ++c) if (rng() % 5 == 0) cs.push_back(c);
            REQUIRE(cuda::extract_rows(t, rs) == extract_rows(t, rs));
            REQUIRE(cuda::extract_cols(t, cs) == extract_cols(t, cs));
        }
        const EndorTensor t = compress(random_dense(6, 9, Dtype::F16, 3, 0.5));
        const std::vector<std::size_t> oob{1, 6}, dup{2, 2}, oobc{0, 9}, uns{5, 1};
        REQUIRE(throws_as<BoundsError>([&] { cuda::extract_rows(t, oob); }));
        REQUIRE(throws_as<std::invalid_argument>([&] { cuda::extract_rows(t, dup); }));
        REQUIRE(throws_as<BoundsError>([&] { cuda::extract_cols(t, oobc); }));
        REQUIRE(throws_as<std::invalid_argument>([&] { cuda::extract_cols(t, uns); }));
    });
    run("quantize_values / dequantize_values bit-exact (test_codec.cpp:324-387)", [] {
        std::mt19937_64 rng(5);
        for (int iter = 0; iter < 30; ++iter) {
            const DenseMatrix w = random_dense(1 + rng() % 50, 1 + rng() % 200, Dtype::F16, rng(),
                                               static_cast<double>(rng() % 101) / 100.0);
            const EndorTensor t = compress(w);
            const EndorTensor qr = quantize_values(t), qc = cuda::quantize_values(t);
            REQUIRE(qc.quant_scale() && *qc.quant_scale() == *qr.quant_scale());
            REQUIRE(std::equal(qc.values().begin(), qc.values().end(), qr.values().begin(), qr.values().end()));
            const EndorTensor dr = dequantize_values(qr), dc = cuda::dequantize_values(qr);
            REQUIRE(std::equal(dc.values().begin(), dc.values().end(), dr.values().begin(), dr.values().end()));
            REQUIRE(cuda::decompress(dc) == decompress(dr));
        }
        REQUIRE(throws_as<std::invalid_argument>([] {
            cuda::quantize_values(compress(random_dense(2, 2, Dtype::I8, 1, 0.0)));
        }));
        REQUIRE(throws_as<std::invalid_argument>([] {
            cuda::dequantize_values(compress(random_dense(2, 2, Dtype::F16, 1, 0.0)));
        }));
    });
    std::printf("%d failure(s)\n", g_fail);
    return g_fail;
}
