// offload_layer.cpp -- what an inference runtime written in C++ does with the
// C ABI: keep a layer's compressed weights in pinned host memory and, per
// token, stream them over PCIe while the GPU computes y = W x for each op
// straight from the compressed form (H2D of op i+1 overlaps op i).
//
//   g++ -std=c++17 -O2 -I include -I /usr/local/cuda/include examples/offload_layer.cpp
//       -L paper_2406_11674_b200 -lendor_cuda -Wl,-rpath,$PWD/paper_2406_11674_b200
//       -L /usr/local/cuda/lib64 -lcudart -o examples/offload_layer
//   examples/offload_layer     # one synthetic OPT-66B-shaped fc1 op, timed
// (tests/test_gpu_example.py builds and runs it)
//
// Weights come from the library's own fixtures (the reference's synth_weight +
// magnitude_prune, weight_gen.hpp:40-113) so the example needs no files.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "endor_cuda.h"

#define CHECK(x)                                                                        \
    do {                                                                                \
        const int st_ = (x);                                                            \
        if (st_) {                                                                      \
            std::fprintf(stderr, "%s failed: %d (%s)\n", #x, st_, endor_cuda_last_error_string()); \
            std::exit(1);                                                               \
        }                                                                               \
    } while (0)

int main() {
    const uint64_t rows = 9216, cols = 36864, n = rows * cols;  // OPT-66B fc1
    void* stream = nullptr;                                      // the default stream
    // 1. fixture weights on the device, pruned to 50 %, compressed (offline in practice)
    void *w, *bm, *vals, *ws;
    cudaMalloc(&w, n * 2);
    cudaMalloc(&bm, (n + 7) / 8 + 16);
    cudaMalloc(&vals, n * 2);
    const size_t ws_bytes = endor_cuda_workspace_bytes(rows, cols);
    cudaMalloc(&ws, ws_bytes);
    CHECK(endor_cuda_workspace_init(ws, ws_bytes, stream));
    CHECK(endor_cuda_synth_weight(rows, cols, ENDOR_DTYPE_F16, 7, 0, rows, w, stream));
    CHECK(endor_cuda_magnitude_prune(n, ENDOR_DTYPE_F16, 0.5, w, ws, ws_bytes, stream));
    uint64_t nnz = 0;
    int32_t negzero = 0;
    CHECK(endor_cuda_compress(rows, cols, ENDOR_DTYPE_F16, w, bm, vals, &nnz, &negzero, ws, ws_bytes, stream));
    // 2. the compressed form moves to pinned host memory: this is what stays resident
    void* h_bm = endor_host_alloc((n + 7) / 8);
    void* h_vals = endor_host_alloc(nnz * 2);
    cudaMemcpy(h_bm, bm, (n + 7) / 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h_vals, vals, nnz * 2, cudaMemcpyDeviceToHost);
    // 3. per token: x on the device, y back on the host
    std::vector<uint16_t> hx(cols, 0x3C00);  // x = 1.0 (f16)
    void* d_x;
    float* d_y;
    cudaMalloc(&d_x, cols * 2);
    cudaMalloc(reinterpret_cast<void**>(&d_y), rows * 4);
    cudaMemcpy(d_x, hx.data(), cols * 2, cudaMemcpyHostToDevice);
    float* h_y = static_cast<float*>(endor_host_alloc(rows * 4));
    endor_pipeline* p;
    CHECK(endor_pipeline_create(0, n, 2, &p));
    endor_pipeline_op op{};
    op.rows = rows;
    op.cols = cols;
    op.dtype = ENDOR_DTYPE_F16;
    op.bitmap_host = h_bm;
    op.values_host = h_vals;
    op.nnz = nnz;
    op.x_dev = d_x;
    op.y_dev = d_y;
    op.y_host = h_y;  // dense_dev NULL: the fused decompress -> GEMV, W never in HBM
    CHECK(endor_pipeline_run(p, &op, 1, 1));  // warm-up
    const auto t0 = std::chrono::steady_clock::now();
    CHECK(endor_pipeline_run(p, &op, 1, 1));
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    endor_pipeline_stats s;
    CHECK(endor_pipeline_stats_get(p, &s));
    std::printf("fc1 %llux%llu @50%%: %.2f ms per offloaded op (H2D %.1f GB/s), y[0] = %f\n",
                (unsigned long long)rows, (unsigned long long)cols, ms,
                s.h2d_bytes / (s.h2d_ms * 1e-3) / 1e9, h_y[0]);
    CHECK(endor_pipeline_destroy(p));
    endor_host_free(h_bm);
    endor_host_free(h_vals);
    endor_host_free(h_y);
    return 0;
}
