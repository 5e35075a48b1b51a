// launch_probe.cu -- measurement aid: how long does a persistent grid take to
// get all of its CTAs running, as a function of dynamic shared memory per CTA?
// Each CTA records %globaltimer at entry; the spread (last start - first
// start) and the event-timed duration of a near-empty kernel are printed.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_probe launch_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

__global__ void probe(unsigned long long* t0, unsigned long long* t1, int spin_ns) {
    extern __shared__ uint8_t smem[];
    unsigned long long a;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a));
    if (threadIdx.x == 0 && spin_ns < 0) smem[0] = 1;  // never: keeps the smem declaration
    unsigned long long b = a;
    while (b - a < (unsigned long long)spin_ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(b));
    __syncthreads();
    if (threadIdx.x == 0) {
        t0[blockIdx.x] = a;
        t1[blockIdx.x] = b;
    }
}

__global__ void fill(uint8_t* p, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) p[i] = uint8_t(i);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *t0, *t1;
    cudaMalloc(&t0, 8 * 4096);
    cudaMalloc(&t1, 8 * 4096);
    uint8_t* scratch;
    const size_t sn = size_t(512) << 20;
    cudaMalloc(&scratch, sn);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Cfg { int ctas_per_sm, threads, smem_kb, spin_ns, flush; };
    const Cfg cfgs[] = {{2, 288, 106, 0, 0}, {2, 288, 106, 0, 1}, {2, 288, 0, 0, 0}, {2, 288, 0, 0, 1},
                        {3, 256, 64, 0, 0},  {3, 256, 64, 0, 1},  {2, 288, 106, 10000, 0}, {2, 288, 106, 10000, 1},
                        {1, 288, 200, 0, 0}, {1, 288, 200, 0, 1}};
    for (const Cfg& c : cfgs) {
        const int grid = c.ctas_per_sm * sms;
        const size_t smem = size_t(c.smem_kb) * 1024;
        std::vector<float> ev;
        std::vector<double> spread, life;
        for (int rep = 0; rep < 12; ++rep) {
            if (c.flush) fill<<<1024, 256>>>(scratch, sn);
            cudaEventRecord(e0);
            probe<<<grid, c.threads, smem>>>(t0, t1, c.spin_ns);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            std::vector<unsigned long long> a(grid), b(grid);
            cudaMemcpy(a.data(), t0, 8 * grid, cudaMemcpyDeviceToHost);
            cudaMemcpy(b.data(), t1, 8 * grid, cudaMemcpyDeviceToHost);
            if (rep < 2) continue;
            ev.push_back(ms * 1000.f);
            const auto mn = *std::min_element(a.begin(), a.end()), mx = *std::max_element(a.begin(), a.end());
            spread.push_back((mx - mn) / 1000.0);
            life.push_back((*std::max_element(b.begin(), b.end()) - mn) / 1000.0);
        }
        std::sort(ev.begin(), ev.end());
        std::sort(spread.begin(), spread.end());
        std::sort(life.begin(), life.end());
        printf("{\"ctas_per_sm\": %d, \"threads\": %d, \"smem_kb\": %d, \"spin_us\": %.1f, \"after_fill\": %d, "
               "\"event_us_median\": %.2f, \"start_spread_us_median\": %.2f, \"first_start_to_last_end_us\": %.2f}\n",
               c.ctas_per_sm, c.threads, c.smem_kb, c.spin_ns / 1000.0, c.flush, ev[ev.size() / 2],
               spread[spread.size() / 2], life[life.size() / 2]);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
