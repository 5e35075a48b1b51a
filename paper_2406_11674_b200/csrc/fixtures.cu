// fixtures.cu -- the reference's input producers on the GPU, bit-exact.
//
//   synth_kernel     synth_weight        weight_gen.hpp:40-55 (SplitMix64 is
//                    counter-based: draw k of seed s is mix(s + k*golden), so
//                    every element is independent)
//   hist/threshold/ties/prune kernels
//                    magnitude_prune     weight_gen.hpp:96-113: the floor(s*n)
//                    smallest elements under (|v| key, index) are zeroed; found
//                    as a key histogram threshold plus an in-order tie cut
//   bitmap/compact kernels
//                    compress            codec.hpp:97-126 (row-major scan,
//                    f16 zero iff (h & 0x7FFF) == 0, -0 flagged)
//
// The paper compresses offline; these exist so the benchmark
// and the full-size parity tests can regenerate the BASELINE.json inputs in
// milliseconds instead of minutes of CPU time.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace endor_b200 {

__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t k) {
    uint64_t z = seed + k * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// next_signed_unit (weight_gen.hpp:29-32), explicit IEEE ops (no contraction)
__device__ __forceinline__ double signed_unit(uint64_t r) {
    const double u = __dmul_rn(double(r >> 11), 0x1.0p-53);
    return __dsub_rn(__dmul_rn(2.0, u), 1.0);
}

template <int EB>
__global__ void synth_kernel(uint64_t i0, uint64_t count, uint64_t seed, uint8_t* out) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < count; t += stride) {
        const double s = signed_unit(splitmix_at(seed, i0 + t + 1));
        if constexpr (EB == 2) {
            reinterpret_cast<uint16_t*>(out)[t] = f32_to_f16_bits(__double2float_rn(s));
        } else {
            long long v = llround(__dmul_rn(s, 127.0));
            v = v < -127 ? -127 : (v > 127 ? 127 : v);
            out[t] = uint8_t(int8_t(v));
        }
    }
}

// ---- magnitude_prune ----------------------------------------------------------
template <int EB>
__device__ __forceinline__ uint32_t mag_key(const uint8_t* w, uint64_t i) {  // weight_gen.hpp:61-64
    if constexpr (EB == 2) return reinterpret_cast<const uint16_t*>(w)[i] & 0x7FFFu;
    const int v = int8_t(w[i]);
    return uint32_t(v < 0 ? -v : v);
}

constexpr int kHistBins = 32768;

template <int EB>
__global__ void __launch_bounds__(1024) hist_kernel(const uint8_t* w, uint64_t n,
                                                    unsigned long long* ghist) {
    extern __shared__ uint32_t sh[];
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        atomicAdd(&sh[mag_key<EB>(w, i)], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
        if (sh[i]) atomicAdd(&ghist[i], (unsigned long long)sh[i]);
}

// One CTA: K = smallest key with cum(<=K) >= target; below = cum(<K).
// Results in hdr->aux[0] (K) and hdr->aux[1] (ties to prune = target-below).
__global__ void __launch_bounds__(1024) threshold_kernel(const unsigned long long* ghist,
                                                         uint64_t target, WsHeader* hdr) {
    constexpr int PER = kHistBins / 1024;
    __shared__ unsigned long long s_tot[1024];
    const int t = threadIdx.x;
    unsigned long long sum = 0;
    for (int j = 0; j < PER; ++j) sum += ghist[t * PER + j];
    s_tot[t] = sum;
    __syncthreads();
    if (t == 0) {  // 1024-entry serial scan, negligible next to the histogram
        unsigned long long run = 0;
        for (int i = 0; i < 1024; ++i) {
            const unsigned long long v = s_tot[i];
            s_tot[i] = run;
            run += v;
        }
    }
    __syncthreads();
    unsigned long long below = s_tot[t];
    if (below < target && below + sum >= target) {
        for (int j = 0; j < PER; ++j) {
            const unsigned long long h = ghist[t * PER + j];
            if (below + h >= target) {
                hdr->aux[0] = uint64_t(t * PER + j);
                hdr->aux[1] = target - below;
                break;
            }
            below += h;
        }
    }
}

// Per-tile count of elements whose key equals K.
template <int EB>
__global__ void __launch_bounds__(256) tie_count_kernel(const uint8_t* w, uint64_t n,
                                                        const WsHeader* hdr,
                                                        unsigned long long* ties) {
    __shared__ uint32_t s_cnt[8];
    const uint32_t K = uint32_t(hdr->aux[0]);
    const uint64_t t0 = uint64_t(blockIdx.x) * kTileElems;
    uint32_t c = 0;
    for (uint32_t j = threadIdx.x; j < kTileElems; j += 256) {
        const uint64_t i = t0 + j;
        if (i < n && mag_key<EB>(w, i) == K) ++c;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
    if ((threadIdx.x & 31) == 0) s_cnt[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int i = 0; i < 8; ++i) s += s_cnt[i];
        ties[blockIdx.x] = s;
    }
}

// Single-CTA exclusive scan of m u64 counters in place (m ~ 1e4-1e5).
__global__ void __launch_bounds__(1024) small_scan_kernel(unsigned long long* v, uint64_t m) {
    __shared__ unsigned long long s_tot[1024];
    const int t = threadIdx.x;
    const uint64_t per = (m + 1023) / 1024;
    const uint64_t b = uint64_t(t) * per, e = min(m, b + per);
    unsigned long long sum = 0;
    for (uint64_t i = b; i < e; ++i) sum += v[i];
    s_tot[t] = sum;
    __syncthreads();
    if (t == 0) {
        unsigned long long run = 0;
        for (int i = 0; i < 1024; ++i) {
            const unsigned long long x = s_tot[i];
            s_tot[i] = run;
            run += x;
        }
    }
    __syncthreads();
    unsigned long long run = s_tot[t];
    for (uint64_t i = b; i < e; ++i) {
        const unsigned long long x = v[i];
        v[i] = run;
        run += x;
    }
}

// Zero key < K, and the first `ties` key == K elements in index order.
template <int EB>
__global__ void __launch_bounds__(256) prune_apply_kernel(uint8_t* w, uint64_t n, const WsHeader* hdr,
                                                          const unsigned long long* ties_prefix) {
    __shared__ uint32_t s_warp[8];
    const uint32_t K = uint32_t(hdr->aux[0]);
    const uint64_t cut = hdr->aux[1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t base = uint64_t(blockIdx.x) * kTileElems + uint64_t(tid) * 32;
    uint32_t eq = 0;
    for (int j = 0; j < 32; ++j) {
        const uint64_t i = base + j;
        if (i < n && mag_key<EB>(w, i) == K) eq |= 1u << j;
    }
    const uint32_t pc = __popc(eq);
    const uint32_t incl = warp_incl_scan(pc, lane);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t wex = 0;
    for (int i = 0; i < warp; ++i) wex += s_warp[i];
    uint64_t rank = ties_prefix[blockIdx.x] + wex + incl - pc;
    for (int j = 0; j < 32; ++j) {
        const uint64_t i = base + j;
        if (i >= n) break;
        const uint32_t k = mag_key<EB>(w, i);
        bool prune = k < K;
        if (eq & (1u << j)) {
            prune = rank < cut;
            ++rank;
        }
        if (prune) {
            if constexpr (EB == 2) reinterpret_cast<uint16_t*>(w)[i] = 0;
            else w[i] = 0;
        }
    }
}

// ---- compress ----------------------------------------------------------------------
// Each thread builds one u32 bitmap word (32 elements).
template <int EB>
__global__ void __launch_bounds__(256) bitmap_kernel(const uint8_t* dense, uint64_t n, uint8_t* bitmap,
                                                     WsHeader* hdr) {
    const uint64_t nwords = (n + 31) / 32;
    const uint64_t nbytes = (n + 7) / 8;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    bool negzero = false;
    for (uint64_t wi = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; wi < nwords; wi += stride) {
        uint32_t word = 0;
        for (int j = 0; j < 32; ++j) {
            const uint64_t i = wi * 32 + j;
            if (i >= n) break;
            bool nz;
            if constexpr (EB == 2) {
                const uint16_t h = reinterpret_cast<const uint16_t*>(dense)[i];
                nz = (h & 0x7FFFu) != 0;  // float16.hpp:75
                negzero |= (h == 0x8000u);
            } else {
                nz = dense[i] != 0;
            }
            word |= uint32_t(nz) << j;
        }
        if (wi * 4 + 4 <= nbytes) {
            reinterpret_cast<uint32_t*>(bitmap)[wi] = word;
        } else {
            for (int b = 0; b < 4; ++b)
                if (wi * 4 + b < nbytes) bitmap[wi * 4 + b] = uint8_t(word >> (8 * b));
        }
    }
    if (negzero) hdr->aux[2] = 1;
}

template <int EB>
__global__ void __launch_bounds__(256) compact_kernel(const uint8_t* dense, uint64_t n,
                                                      const uint8_t* bitmap, uint64_t nbytes,
                                                      const unsigned long long* tprefix,
                                                      uint8_t* values) {
    __shared__ uint32_t s_warp[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t wi = uint64_t(blockIdx.x) * kTileWords + tid;
    const uint32_t word = (wi * 32 < n) ? load_word32(bitmap, wi, nbytes) : 0u;
    const uint32_t pc = __popc(word);
    const uint32_t incl = warp_incl_scan(pc, lane);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t wex = 0;
    for (int i = 0; i < warp; ++i) wex += s_warp[i];
    uint64_t v = tprefix[blockIdx.x] + wex + incl - pc;
    uint32_t m = word;
    while (m) {
        const int j = __ffs(m) - 1;
        const uint64_t i = wi * 32 + j;
        if constexpr (EB == 2) {
            const uint16_t h = reinterpret_cast<const uint16_t*>(dense)[i];
            values[2 * v] = uint8_t(h);
            values[2 * v + 1] = uint8_t(h >> 8);
        } else {
            values[v] = dense[i];
        }
        ++v;
        m &= m - 1;
    }
}

// ---- compress, vectorised (16-byte aligned dense input) -----------------------
// The same predicate as bitmap_kernel / compact_kernel (f16 zero iff
// (h & 0x7FFF) == 0, float16.hpp:75; i8 zero iff 0), but coalesced: a thread
// owns 16-byte chunks (8 f16 / 16 i8 elements).  bitmap: one mask byte (or
// two) per chunk.  compact: CTA per 8192-element tile, the chunk masks are
// recomputed from the data, one block scan places every chunk's values, the
// tile's packed values are staged in shared memory at the destination's
// 16-byte phase and leave with 16-byte stores.
template <int EB>
__device__ __forceinline__ uint32_t chunk_mask(const uint4 v, bool& negzero) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t m = 0;
    if constexpr (EB == 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t h = (w[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
            m |= uint32_t((h & 0x7FFFu) != 0) << k;
            negzero |= h == 0x8000u;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) m |= uint32_t(((w[k >> 2] >> (8 * (k & 3))) & 0xFFu) != 0) << k;
    }
    return m;
}

template <int EB>
__global__ void __launch_bounds__(256) bitmap_vec_kernel(const uint4* __restrict__ dense, uint64_t n,
                                                         uint8_t* __restrict__ bitmap, WsHeader* hdr) {
    constexpr int EPC = 16 / EB;
    const uint64_t nfull = n / EPC, nbytes = (n + 7) / 8;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    bool negzero = false;
    for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < nfull; c += stride) {
        const uint32_t m = chunk_mask<EB>(__ldcs(dense + c), negzero);
        if constexpr (EB == 2) bitmap[c] = uint8_t(m);
        else reinterpret_cast<uint16_t*>(bitmap)[c] = uint16_t(m);  // bitmap is 4-byte aligned
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && nfull * EPC < n) {  // the ragged last chunk, elementwise
        const uint8_t* d = reinterpret_cast<const uint8_t*>(dense);
        uint32_t m = 0;
        for (uint64_t i = nfull * EPC; i < n; ++i) {
            bool nz;
            if constexpr (EB == 2) {
                const uint16_t h = reinterpret_cast<const uint16_t*>(d)[i];
                nz = (h & 0x7FFFu) != 0;
                negzero |= h == 0x8000u;
            } else {
                nz = d[i] != 0;
            }
            m |= uint32_t(nz) << (i - nfull * EPC);
        }
        for (uint64_t b = nfull * EPC / 8; b < nbytes; ++b) bitmap[b] = uint8_t(m >> (8 * (b - nfull * EPC / 8)));
    }
    if (negzero) hdr->aux[2] = 1;
}

template <int EB>
__global__ void __launch_bounds__(256) compact_vec_kernel(const uint4* __restrict__ dense, uint64_t n,
                                                          const unsigned long long* __restrict__ tprefix,
                                                          uint8_t* __restrict__ values) {
    constexpr int EPC = 16 / EB, CPT = kTileElems / EPC / 256;  // chunks per thread (consecutive)
    __shared__ __align__(16) uint8_t s_out[kTileElems * EB + 16];
    __shared__ uint32_t s_warp[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t c0 = uint64_t(blockIdx.x) * (kTileElems / EPC) + uint64_t(tid) * CPT;  // first chunk
    uint4 v[CPT];
    uint32_t m[CPT], cnt = 0;
    bool nz0 = false;
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
        const uint64_t e0 = (c0 + r) * EPC;
        v[r] = make_uint4(0, 0, 0, 0);
        if (e0 + EPC <= n) {
            v[r] = __ldcs(dense + c0 + r);
        } else if (e0 < n) {  // the ragged last chunk: only the elements inside the matrix
            uint32_t w[4] = {0, 0, 0, 0};
            const uint8_t* d = reinterpret_cast<const uint8_t*>(dense);
            for (uint64_t i = e0; i < n; ++i) w[((i - e0) * EB) >> 2] |= uint32_t(d[i * EB]) << (8 * (((i - e0) * EB) & 3)) |
                                                                   (EB == 2 ? uint32_t(d[i * EB + 1]) << (8 * (((i - e0) * EB + 1) & 3)) : 0u);
            v[r] = make_uint4(w[0], w[1], w[2], w[3]);
        }
        m[r] = chunk_mask<EB>(v[r], nz0);
        cnt += __popc(m[r]);
    }
    const uint32_t incl = warp_incl_scan(cnt, lane);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t base = 0, total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        base += w < warp ? s_warp[w] : 0u;
        total += s_warp[w];
    }
    uint8_t* dst = values + tprefix[blockIdx.x] * EB;
    const uint32_t ph = uint32_t(reinterpret_cast<uintptr_t>(dst) & 15);  // stage at the destination's phase
    uint32_t pos = base + incl - cnt;
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
        const uint32_t w[4] = {v[r].x, v[r].y, v[r].z, v[r].w};
#pragma unroll
        for (int k = 0; k < EPC; ++k) {
            if ((m[r] >> k) & 1u) {
                if constexpr (EB == 2) {
                    *reinterpret_cast<uint16_t*>(s_out + ph + 2 * pos) = uint16_t(w[k >> 1] >> (16 * (k & 1)));
                } else {
                    s_out[ph + pos] = uint8_t(w[k >> 2] >> (8 * (k & 3)));
                }
                ++pos;
            }
        }
    }
    __syncthreads();
    const uint32_t bytes = total * EB, head = (16 - ph) & 15;
    if (bytes <= head) {
        for (uint32_t b = tid; b < bytes; b += 256) dst[b] = s_out[ph + b];
        return;
    }
    for (uint32_t b = tid; b < head; b += 256) dst[b] = s_out[ph + b];
    const uint32_t nvec = (bytes - head) / 16;
    const uint4* src4 = reinterpret_cast<const uint4*>(s_out + ph + head);
    uint4* dst4 = reinterpret_cast<uint4*>(dst + head);
    for (uint32_t q = tid; q < nvec; q += 256) dst4[q] = src4[q];
    for (uint32_t b = head + nvec * 16 + tid; b < bytes; b += 256) dst[b] = s_out[ph + b];
}

// ---- quantize_values (codec.hpp:306-331) ---------------------------------------
// absmax over |f16_to_f32(v)| (NaNs never win, like std::max(absmax, x)),
// then q = clamp(lround(v / scale), -127, 127) with IEEE float division.
__device__ __forceinline__ float f16_bits_to_f32(uint16_t h) { return __half2float(__ushort_as_half(h)); }

__global__ void __launch_bounds__(256) absmax_kernel(const uint16_t* v, uint64_t nnz, unsigned int* amax_bits) {
    float m = 0.f;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nnz; i += stride) {
        const float a = fabsf(f16_bits_to_f32(v[i]));
        m = (m < a) ? a : m;  // a NaN is never selected
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const float o = __shfl_xor_sync(0xffffffffu, m, d);
        m = (m < o) ? o : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(amax_bits, __float_as_uint(m));  // non-negative floats order as ints
}

__global__ void __launch_bounds__(256) quantize_kernel(const uint16_t* v, uint64_t nnz, const unsigned int* amax_bits,
                                                       int8_t* q, float* scale_out) {
    const float absmax = __uint_as_float(*amax_bits);
    const float scale = (nnz == 0 || absmax == 0.0f) ? 1.0f : __fdiv_rn(absmax, 127.0f);
    if (blockIdx.x == 0 && threadIdx.x == 0) *scale_out = scale;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nnz; i += stride) {
        const float x = __fdiv_rn(f16_bits_to_f32(v[i]), scale);
        // x86-64 lround gives the "integer indefinite" LONG_MIN for NaN / out of range
        long long r = (isfinite(x) && fabsf(x) < 9.2e18f) ? llroundf(x) : (-0x7fffffffffffffffll - 1);
        r = r < -127 ? -127 : (r > 127 ? 127 : r);
        q[i] = int8_t(r);
    }
}

cudaError_t launch_quantize(const void* vals, uint64_t nnz, void* q, float* scale_dev, unsigned int* amax,
                            cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(amax, 0, sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
    const unsigned g = unsigned(nnz ? (ceil_div(nnz, 256) < 148 * 16 ? ceil_div(nnz, 256) : 148 * 16) : 1);
    absmax_kernel<<<g, 256, 0, s>>>(static_cast<const uint16_t*>(vals), nnz, amax);
    quantize_kernel<<<g, 256, 0, s>>>(static_cast<const uint16_t*>(vals), nnz, amax, static_cast<int8_t*>(q),
                                      scale_dev);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static unsigned grid_for(uint64_t work, unsigned threads, unsigned cap = 148 * 32) {
    const uint64_t g = ceil_div(work, threads);
    return unsigned(g < 1 ? 1 : (g > cap ? cap : g));
}

// dequantize_values (codec.hpp:334-349): f16 = f32_to_f16(float(q) * scale)
// per packed value, RNE (float16.hpp:35-73); NaN products follow the x86 SSE
// rules the reference runs under (see gather_chunk_dequant).
__global__ void __launch_bounds__(256) dequant_values_kernel(const int8_t* q, uint64_t nnz, float scale,
                                                             uint16_t* out) {
    const uint32_t sb = __float_as_uint(scale);
    const bool snan = (sb & 0x7FFFFFFFu) > 0x7F800000u;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nnz; i += uint64_t(gridDim.x) * blockDim.x) {
        float v = __fmul_rn(float(q[i]), scale);
        if (v != v) v = __uint_as_float(snan ? (sb | 0x00400000u) : 0xFFC00000u);
        out[i] = f32_to_f16_bits(v);
    }
}

cudaError_t launch_dequant_values(const void* q, uint64_t nnz, float scale, void* out, cudaStream_t s) {
    if (nnz == 0) return cudaSuccess;
    const unsigned g = unsigned(umin64(ceil_div(nnz, 256), 148ull * 16));
    dequant_values_kernel<<<g, 256, 0, s>>>(static_cast<const int8_t*>(q), nnz, scale, static_cast<uint16_t*>(out));
    return cudaGetLastError();
}

cudaError_t launch_synth(uint64_t i0, uint64_t count, int eb, uint64_t seed, void* out,
                         cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    const unsigned g = grid_for(count, 256);
    if (eb == 2) synth_kernel<2><<<g, 256, 0, s>>>(i0, count, seed, static_cast<uint8_t*>(out));
    else synth_kernel<1><<<g, 256, 0, s>>>(i0, count, seed, static_cast<uint8_t*>(out));
    return cudaGetLastError();
}

cudaError_t launch_prune(uint8_t* w, uint64_t n, int eb, uint64_t target, const WsLayout& L,
                         cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(L.hist, 0, sizeof(unsigned long long) * kHistBins, s);
    if (e != cudaSuccess) return e;
    const size_t smem = sizeof(uint32_t) * kHistBins;
    int sms = 148;
    e = kernel_slots(eb == 2 ? reinterpret_cast<const void*>(hist_kernel<2>)
                             : reinterpret_cast<const void*>(hist_kernel<1>),
                     1024, smem, nullptr, &sms);
    if (e != cudaSuccess) return e;
    const uint64_t want = ceil_div(n, 1024);
    const unsigned hg = unsigned(want < uint64_t(sms) ? want : uint64_t(sms));
    if (eb == 2) hist_kernel<2><<<hg, 1024, smem, s>>>(w, n, L.hist);
    else hist_kernel<1><<<hg, 1024, smem, s>>>(w, n, L.hist);
    threshold_kernel<<<1, 1024, 0, s>>>(L.hist, target, L.hdr);
    const unsigned nt = unsigned(ceil_div(n, kTileElems));
    if (eb == 2) tie_count_kernel<2><<<nt, 256, 0, s>>>(w, n, L.hdr, L.ties);
    else tie_count_kernel<1><<<nt, 256, 0, s>>>(w, n, L.hdr, L.ties);
    small_scan_kernel<<<1, 1024, 0, s>>>(L.ties, nt);
    if (eb == 2) prune_apply_kernel<2><<<nt, 256, 0, s>>>(w, n, L.hdr, L.ties);
    else prune_apply_kernel<1><<<nt, 256, 0, s>>>(w, n, L.hdr, L.ties);
    return cudaGetLastError();
}

cudaError_t launch_bitmap(const void* dense, uint64_t n, int eb, void* bitmap, const WsLayout& L,
                          cudaStream_t s) {
    if ((reinterpret_cast<uintptr_t>(dense) & 15) == 0) {  // coalesced 16-byte chunks
        const unsigned g = grid_for(ceil_div(n, 16 / eb), 256);
        if (eb == 2) bitmap_vec_kernel<2><<<g, 256, 0, s>>>(static_cast<const uint4*>(dense), n, static_cast<uint8_t*>(bitmap), L.hdr);
        else bitmap_vec_kernel<1><<<g, 256, 0, s>>>(static_cast<const uint4*>(dense), n, static_cast<uint8_t*>(bitmap), L.hdr);
        return cudaGetLastError();
    }
    const unsigned g = grid_for(ceil_div(n, 32), 256);
    if (eb == 2) bitmap_kernel<2><<<g, 256, 0, s>>>(static_cast<const uint8_t*>(dense), n, static_cast<uint8_t*>(bitmap), L.hdr);
    else bitmap_kernel<1><<<g, 256, 0, s>>>(static_cast<const uint8_t*>(dense), n, static_cast<uint8_t*>(bitmap), L.hdr);
    return cudaGetLastError();
}

cudaError_t launch_compact(const void* dense, uint64_t n, int eb, const void* bitmap,
                           const WsLayout& L, void* values, cudaStream_t s) {
    const unsigned nt = unsigned(ceil_div(n, kTileElems));
    if (nt == 0) return cudaSuccess;
    if ((reinterpret_cast<uintptr_t>(dense) & 15) == 0) {  // coalesced 16-byte chunks, staged 16-byte stores
        if (eb == 2) compact_vec_kernel<2><<<nt, 256, 0, s>>>(static_cast<const uint4*>(dense), n, L.tprefix, static_cast<uint8_t*>(values));
        else compact_vec_kernel<1><<<nt, 256, 0, s>>>(static_cast<const uint4*>(dense), n, L.tprefix, static_cast<uint8_t*>(values));
        return cudaGetLastError();
    }
    const uint64_t nbytes = (n + 7) / 8;
    if (eb == 2)
        compact_kernel<2><<<nt, 256, 0, s>>>(static_cast<const uint8_t*>(dense), n, static_cast<const uint8_t*>(bitmap), nbytes, L.tprefix, static_cast<uint8_t*>(values));
    else
        compact_kernel<1><<<nt, 256, 0, s>>>(static_cast<const uint8_t*>(dense), n, static_cast<const uint8_t*>(bitmap), nbytes, L.tprefix, static_cast<uint8_t*>(values));
    return cudaGetLastError();
}

}  // namespace endor_b200
