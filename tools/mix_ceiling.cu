// Practical HBM ceiling for the decompress's read/write mix (development aid):
// a streaming kernel that reads 9 and writes 16 16-byte vectors per 16 output
// vectors (read/write = 0.5625 = (1/8 + 1) / 2 for f16 @ 50 %), no math.
#include <cuda_runtime.h>
#include <stdint.h>
__global__ void mix_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, uint64_t nout) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nout; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t g = i >> 4, r = i & 15;
        uint4 v = make_uint4(uint32_t(i), 0, 0, 0);
        if (r < 9) v = __ldcs(src + g * 9 + r);
        __stcs(dst + i, v);
    }
}
__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, uint64_t n) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        __stcs(dst + i, __ldcs(src + i));
}
extern "C" float mix_time(const void* src, void* dst, uint64_t nout_vec, int reps, int which, int blocks) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int k = 0; k < reps + 2; ++k) {
        if (k == 2) cudaEventRecord(a);
        if (which == 0) mix_kernel<<<blocks, 512>>>((const uint4*)src, (uint4*)dst, nout_vec);
        else copy_kernel<<<blocks, 512>>>((const uint4*)src, (uint4*)dst, nout_vec);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}
