// Write-path variants for the expand kernel's 9:16 read:write mix (development aid):
//   mode 0: 16-byte st.global (as the expand kernel)
//   mode 1: stage 16 KiB per CTA in smem, then one cp.async.bulk S2G store
//   mode 2: per-warp 2 KiB cp.async.bulk S2G stores
//   mode 3: 32-byte st.global.v8 (sm_100 256-bit stores), .cs
//   mode 4: 32-byte st.global.v8, default policy
//   mode 5: 16-byte st.global (default policy)
//   mode 6: 16-byte st.global.L1::no_allocate
//   mode 7: 16-byte st.global.L2::cache_hint (evict_first policy)
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
template <int MODE>
__global__ void __launch_bounds__(256) mix2(const uint4* __restrict__ src, uint4* __restrict__ dst, uint64_t nblk) {
    __shared__ __align__(128) uint4 buf[2][1024];  // 2 x 16 KiB
    int it = 0;
    for (uint64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++it) {
        const int s = it & 1;
        // each block: 1024 output vectors (16 KiB), 576 input vectors (9/16)
        uint4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t o = MODE == 2 ? (threadIdx.x >> 5) * 128 + (threadIdx.x & 31) + 32 * j
                                         : threadIdx.x + 256 * j;  // output vector within the block
            const uint32_t r = o & 15;
            v[j] = make_uint4(o, 0, 0, 0);
            if (r < 9) v[j] = __ldcs(src + blk * 576 + (o >> 4) * 9 + r);
        }
        if (MODE == 1) {
            if (threadIdx.x == 0 && it >= 2)
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // buf[s] free again
            __syncthreads();
#pragma unroll
            for (int j = 0; j < 4; ++j) buf[s][threadIdx.x + 256 * j] = v[j];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                             ::"l"(dst + blk * 1024), "r"(smem_u32(buf[s])), "r"(16384) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        } else if (MODE == 2) {  // per-warp 2 KiB bulk stores (each warp owns 128 vectors of the block)
            const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
            if (l == 0 && it >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 4; ++j) buf[s][w * 128 + l + 32 * j] = v[j];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (l == 0) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                             ::"l"(dst + blk * 1024 + w * 128), "r"(smem_u32(&buf[s][w * 128])), "r"(2048) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        } else if (MODE == 3 || MODE == 4) {  // 32-byte stores: thread t writes vectors 2t,2t+1 (+512)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                uint4* d = dst + blk * 1024 + 2 * threadIdx.x + 512 * j;
                const uint4 a = v[2 * j], c = v[2 * j + 1];
                if (MODE == 3)
                    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(d), "r"(a.x), "r"(a.y),
                                 "r"(a.z), "r"(a.w), "r"(c.x), "r"(c.y), "r"(c.z), "r"(c.w) : "memory");
                else
                    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(d), "r"(a.x), "r"(a.y),
                                 "r"(a.z), "r"(a.w), "r"(c.x), "r"(c.y), "r"(c.z), "r"(c.w) : "memory");
            }
        } else if (MODE == 5) {
#pragma unroll
            for (int j = 0; j < 4; ++j) dst[blk * 1024 + threadIdx.x + 256 * j] = v[j];
        } else if (MODE == 6) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst + blk * 1024 + threadIdx.x + 256 * j),
                             "r"(v[j].x), "r"(v[j].y), "r"(v[j].z), "r"(v[j].w) : "memory");
        } else if (MODE == 7) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
            for (int j = 0; j < 4; ++j)
                asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(dst + blk * 1024 + threadIdx.x + 256 * j),
                             "r"(v[j].x), "r"(v[j].y), "r"(v[j].z), "r"(v[j].w), "l"(pol) : "memory");
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) __stcs(dst + blk * 1024 + threadIdx.x + 256 * j, v[j]);
        }
    }
    if (MODE == 1 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (MODE == 2 && (threadIdx.x & 31) == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
extern "C" float mix2_time(const void* src, void* dst, uint64_t nblk, int reps, int mode, int blocks) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int k = 0; k < reps + 2; ++k) {
        if (k == 2) cudaEventRecord(a);
        if (mode == 1) mix2<1><<<blocks, 256>>>((const uint4*)src, (uint4*)dst, nblk);
        else if (mode == 2) mix2<2><<<blocks, 256>>>((const uint4*)src, (uint4*)dst, nblk);
        else if (mode == 3) mix2<3><<<blocks, 256>>>((const uint4*)src, (uint4*)dst, nblk);
        else if (mode == 4) mix2<4><<<blocks, 256>>>((const uint4*)src, (uint4*)dst, nblk);
        else if (mode == 5) mix2<5><<<blocks, 256>>>((const uint4*)src, (uint4*)dst, nblk);
        else if (mode == 6) mix2<6><<<blocks, 256>>>((const uint4*)src, (uint4*)dst, nblk);
        else if (mode == 7) mix2<7><<<blocks, 256>>>((const uint4*)src, (uint4*)dst, nblk);
        else mix2<0><<<blocks, 256>>>((const uint4*)src, (uint4*)dst, nblk);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}
