// read_ceiling.cu -- measurement aid: how fast can a kernel READ n bytes on
// this B200 (the count pass's roofline is a pure read stream)?  Plain 16-byte
// loads with popcount accumulation, grid = SMs x k, timed with CUDA events
// back-to-back over rotating buffers (inputs >> L2 in total).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_ceiling read_ceiling.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

template <int U>
__global__ void __launch_bounds__(256) read_popc(const uint4* __restrict__ p, size_t n16, unsigned long long* out) {
    uint32_t c = 0;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    for (; i + (U - 1) * stride < n16; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) c += __popc(v[u].x) + __popc(v[u].y) + __popc(v[u].z) + __popc(v[u].w);
    }
    for (; i < n16; i += stride) {
        const uint4 v = __ldcs(p + i);
        c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    }
    if (c == 0xFFFFFFFFu) atomicAdd(out, c);  // keeps the loads live
}

// contiguous per-CTA ranges (the count kernel's static partition)
template <int U>
__global__ void __launch_bounds__(256) read_popc_ranges(const uint4* __restrict__ p, size_t n16, unsigned long long* out) {
    uint32_t c = 0;
    const size_t per = (n16 + gridDim.x - 1) / gridDim.x;
    const size_t r0 = blockIdx.x * per, r1 = r0 + per < n16 ? r0 + per : n16;
    size_t i = r0 + threadIdx.x;
    for (; i + (U - 1) * blockDim.x < r1; i += U * blockDim.x) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * blockDim.x);
#pragma unroll
        for (int u = 0; u < U; ++u) c += __popc(v[u].x) + __popc(v[u].y) + __popc(v[u].z) + __popc(v[u].w);
    }
    for (; i < r1; i += blockDim.x) {
        const uint4 v = __ldcs(p + i);
        c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    }
    if (c == 0xFFFFFFFFu) atomicAdd(out, c);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t sizes[] = {size_t(4) << 20, size_t(13) << 20, size_t(42) << 20, size_t(127) << 20, size_t(512) << 20};
    const int R = 8;
    uint8_t* buf;
    cudaMalloc(&buf, size_t(R) * (size_t(512) << 20) / 2 + (size_t(512) << 20));
    unsigned long long* out;
    cudaMalloc(&out, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (size_t n : sizes) {
        const int copies = n * R <= (size_t(2) << 30) ? R : 2;
        for (int k : {3, 4, 8}) {
            const size_t n16 = n / 16;
            const int grid = sms * k;
            for (int w = 0; w < 3; ++w) read_popc<4><<<grid, 256>>>(reinterpret_cast<const uint4*>(buf), n16, out);
            cudaEventRecord(a);
            const int reps = 20 * copies;
            for (int r = 0; r < reps; ++r)
                read_popc<4><<<grid, 256>>>(reinterpret_cast<const uint4*>(buf + (r % copies) * n), n16, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            ms /= reps;
            printf("read %8.1f MB  grid %4d: %8.2f us  %7.1f GB/s\n", n / 1e6, grid, ms * 1e3, n / ms / 1e6);
            cudaEventRecord(a);
            for (int r = 0; r < reps; ++r)
                read_popc_ranges<8><<<grid, 256>>>(reinterpret_cast<const uint4*>(buf + (r % copies) * n), n16, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            ms /= reps;
            printf("  ranges %8.1f MB  grid %4d: %8.2f us  %7.1f GB/s\n", n / 1e6, grid, ms * 1e3, n / ms / 1e6);
        }
    }
    return 0;
}
