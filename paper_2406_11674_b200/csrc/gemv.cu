// gemv.cu -- the offloaded op's consumer: y = W x, f16 W [rows, cols]
// row-major (rows = outputs), f16 x, fp32 accumulation.
//
// The reference has no consumer; it models compute as a constant
// (sim.hpp:30,227).  A GEMV at batch 1 is HBM-bound (2 B per weight element,
// 2 FLOP each), so this is a streaming kernel, not a tensor-core GEMM: each
// warp owns R rows, lanes stride the row with 16-byte loads (8 halves) and
// reuse every x vector load across the R rows, then a shuffle reduction.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "gather.cuh"
#include "kernels.h"

namespace endor_b200 {

constexpr int kGemvThreads = 256;

// One launch for a whole batch (a decoder layer's ops): warp g owns R rows of
// tensor k (k found from the per-tensor warp prefix), lanes stride the rows
// with 16-byte streaming loads, U iterations in flight; every x load is
// reused across the R rows.  The f16 x f16 products accumulate in fp32 with
// FHFMA (fma.rn.f32.f16, one instruction per weight).
template <int R, int U>
__global__ void __launch_bounds__(kGemvThreads) gemv_batch_kernel(const __grid_constant__ GemvBatch gb) {
    const int lane = threadIdx.x & 31;
    const uint64_t g = (uint64_t(blockIdx.x) * kGemvThreads + threadIdx.x) >> 5;
    if (g >= gb.warp0[gb.count]) return;
    int k = 0;
    while (g >= gb.warp0[k + 1]) ++k;
    const uint64_t rows = gb.rows[k], cols8 = gb.cols[k] / 8;
    const uint64_t r0 = (g - gb.warp0[k]) * R;
    const uint4* __restrict__ W = static_cast<const uint4*>(gb.w[k]);
    const uint4* __restrict__ x = static_cast<const uint4*>(gb.x[k]);
    const uint4* wr[R];
#pragma unroll
    for (int r = 0; r < R; ++r) wr[r] = W + min(r0 + r, rows - 1) * cols8;
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;
    uint64_t c = lane;
    for (; c + 32 * (U - 1) < cols8; c += 32 * U) {
        uint4 xv[U], wv[U][R];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            xv[u] = __ldg(x + c + 32 * u);
#pragma unroll
            for (int r = 0; r < R; ++r) wv[u][r] = __ldcs(wr[r] + c + 32 * u);  // streamed once: evict-first
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = dot8_f16(wv[u][r], xv[u], acc[r]);
    }
    for (; c < cols8; c += 32) {
        const uint4 xv = __ldg(x + c);
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = dot8_f16(__ldcs(wr[r] + c), xv, acc[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], d);
    }
    if (lane == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (r0 + r < rows) {
                if (gb.y32[k]) gb.y32[k][r0 + r] = acc[r];
                if (gb.y16[k]) static_cast<__half*>(gb.y16[k])[r0 + r] = __float2half_rn(acc[r]);
            }
        }
    }
}

constexpr int kGemvRows = 2, kGemvUnroll = 4;

cudaError_t launch_gemv_batch(GemvBatch& gb, cudaStream_t s) {
    uint64_t warps = 0;
    for (int k = 0; k < gb.count; ++k) {
        gb.warp0[k] = warps;
        warps += ceil_div(gb.rows[k], kGemvRows);
    }
    gb.warp0[gb.count] = warps;
    if (warps == 0) return cudaSuccess;
    const unsigned grid = unsigned(ceil_div(warps * 32, kGemvThreads));
    gemv_batch_kernel<kGemvRows, kGemvUnroll><<<grid, kGemvThreads, 0, s>>>(gb);
    return cudaGetLastError();
}

// Generic (any cols / alignment) path: one warp per row, scalar halves.
__global__ void __launch_bounds__(kGemvThreads) gemv_scalar_kernel(const __half* __restrict__ W,
                                                                    const __half* __restrict__ x,
                                                                    uint64_t rows, uint64_t cols,
                                                                    float* y32, __half* y16) {
    const int lane = threadIdx.x & 31;
    const uint64_t row = (uint64_t(blockIdx.x) * kGemvThreads + threadIdx.x) >> 5;
    if (row >= rows) return;
    float acc = 0.f;
    for (uint64_t c = lane; c < cols; c += 32)
        acc = fmaf(__half2float(W[row * cols + c]), __half2float(x[c]), acc);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
    if (lane == 0) {
        if (y32) y32[row] = acc;
        if (y16) y16[row] = __float2half_rn(acc);
    }
}

cudaError_t launch_gemv(uint64_t rows, uint64_t cols, const void* w, const void* x, float* y32,
                        void* y16, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    const bool vec = (cols % 8 == 0) && ((reinterpret_cast<uintptr_t>(w) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    if (vec) {
        GemvBatch gb{};
        gb.count = 1;
        gb.rows[0] = rows;
        gb.cols[0] = cols;
        gb.w[0] = w;
        gb.x[0] = x;
        gb.y32[0] = y32;
        gb.y16[0] = y16;
        return launch_gemv_batch(gb, s);
    }
    const unsigned grid = unsigned(ceil_div(rows * 32, kGemvThreads));
    gemv_scalar_kernel<<<grid, kGemvThreads, 0, s>>>(static_cast<const __half*>(w), static_cast<const __half*>(x),
                                                      rows, cols, y32, static_cast<__half*>(y16));
    return cudaGetLastError();
}

}  // namespace endor_b200
