// param size probe: empty-ish persistent kernel with small vs 8 KB params
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
struct Big { uint64_t v[1040]; };
__global__ void k_small(uint64_t* out, uint64_t a) { if (threadIdx.x == 0 && blockIdx.x == 9999) out[0] = a; }
__global__ void k_big(uint64_t* out, const __grid_constant__ Big b) { if (threadIdx.x == 0 && blockIdx.x == 9999) out[0] = b.v[blockIdx.x & 1023]; }
__global__ void fill(uint8_t* p, size_t n) { for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) p[i] = uint8_t(i); }
int main() {
  uint64_t* o; cudaMalloc(&o, 64); uint8_t* s; cudaMalloc(&s, 512u<<20);
  Big b{}; cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int smems[3] = {0, 64*1024, 200*1024};
  for (int si = 0; si < 3; ++si) {
    int sm = smems[si];
    cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    for (int grid : {148, 296, 444}) {
      for (int big = 0; big < 2; ++big) {
        float single = 0, b2b = 0;
        for (int rep = 0; rep < 12; ++rep) {
          fill<<<1184, 256>>>(s, 512u<<20);
          cudaEventRecord(e0);
          if (big) k_big<<<grid, 288, sm>>>(o, b); else k_small<<<grid, 288, sm>>>(o, 1);
          cudaEventRecord(e1); cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep >= 2) single += ms / 10;
        }
        cudaEventRecord(e0);
        for (int rep = 0; rep < 100; ++rep) { if (big) k_big<<<grid, 288, sm>>>(o, b); else k_small<<<grid, 288, sm>>>(o, 1); }
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); b2b = ms / 100;
        printf("smem %6d grid %3d params %s: single %.2f us  back-to-back %.2f us\n", sm, grid, big ? "8KB" : "16B", single * 1e3, b2b * 1e3);
      }
    }
  }
  return 0;
}
