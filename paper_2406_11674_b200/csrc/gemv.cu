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
#include "kernels.h"

namespace endor_b200 {

constexpr int kGemvThreads = 256;

__device__ __forceinline__ float dot8(const uint4& w, const uint4& x) {
    const __half2* wh = reinterpret_cast<const __half2*>(&w);
    const __half2* xh = reinterpret_cast<const __half2*>(&x);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 a = __half22float2(wh[i]);
        const float2 b = __half22float2(xh[i]);
        acc = fmaf(a.x, b.x, acc);
        acc = fmaf(a.y, b.y, acc);
    }
    return acc;
}

// cols % 8 == 0 and 16-byte aligned W / x: vector path.
template <int R>
__global__ void __launch_bounds__(kGemvThreads) gemv_vec_kernel(const uint4* __restrict__ W,
                                                                 const uint4* __restrict__ x,
                                                                 uint64_t rows, uint64_t cols8,
                                                                 float* y32, __half* y16) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * kGemvThreads + threadIdx.x) >> 5;
    const uint64_t r0 = warp * R;
    if (r0 >= rows) return;
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;
    const uint4* wr[R];
#pragma unroll
    for (int r = 0; r < R; ++r) wr[r] = W + min(r0 + r, rows - 1) * cols8;
#pragma unroll 2
    for (uint64_t c = lane; c < cols8; c += 32) {
        const uint4 xv = __ldg(x + c);
        uint4 wv[R];
#pragma unroll
        for (int r = 0; r < R; ++r) wv[r] = __ldcs(wr[r] + c);  // streamed once: evict-first
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] += dot8(wv[r], xv);
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
                if (y32) y32[r0 + r] = acc[r];
                if (y16) y16[r0 + r] = __float2half_rn(acc[r]);
            }
        }
    }
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
        constexpr int R = 4;
        const uint64_t warps = ceil_div(rows, R);
        const unsigned grid = unsigned(ceil_div(warps * 32, kGemvThreads));
        gemv_vec_kernel<R><<<grid, kGemvThreads, 0, s>>>(static_cast<const uint4*>(w),
                                                          static_cast<const uint4*>(x), rows,
                                                          cols / 8, y32, static_cast<__half*>(y16));
    } else {
        const unsigned grid = unsigned(ceil_div(rows * 32, kGemvThreads));
        gemv_scalar_kernel<<<grid, kGemvThreads, 0, s>>>(static_cast<const __half*>(w),
                                                          static_cast<const __half*>(x), rows, cols,
                                                          y32, static_cast<__half*>(y16));
    }
    return cudaGetLastError();
}

}  // namespace endor_b200
