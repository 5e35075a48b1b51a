// vcode.cu -- lossless transport coding of the packed f16 values for the
// CpuToGpu stage (no reference counterpart).
//
// The reference's Endor mode is bound by the host -> GPU link: every byte of
// the compressed tensor crosses it (sim.hpp:200-204, bw_cpu_gpu at
// sim.hpp:322-325), and here the pipeline already runs the copy at the pinned
// peak.  The only lever left on that stage is fewer bytes.  A magnitude-pruned
// f16 weight keeps |w| above the pruning threshold, so the high byte of a
// surviving value (sign, 5 exponent bits, top 2 mantissa bits) takes few
// distinct values, while the low byte is noise.  The blob keeps the low bytes
// raw and codes the high byte in k bits through a dictionary of the 2^k - 1
// most frequent high bytes (code 2^k - 1 = exception, listed separately); k is
// chosen per tensor to minimise the blob.  Decoding is one pass with no
// serial dependency (value i's code sits at bit k*i), then a patch pass over
// the exceptions, and reproduces the values bit for bit.
//
// Blob layout: see endor_vcode_header in include/endor_cuda.h.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "endor_cuda.h"
#include "kernels.h"

using namespace endor_b200;

namespace {

constexpr uint32_t kMagic = 0x31435645u;  // "EVC1"
constexpr int kMaxK = 7;
static_assert(sizeof(endor_vcode_header) == 256, "blob header is 256 bytes");

uint64_t up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

// section offsets of a blob for (nnz, k, n_exc)
void layout(uint64_t nnz, uint32_t k, uint64_t n_exc, endor_vcode_header* h) {
    h->lo_off = sizeof(endor_vcode_header);
    h->code_off = h->lo_off + up(nnz, 32);
    h->exc_off = h->code_off + up((nnz + 31) / 32 * k * 4, 16);
    h->blob_bytes = h->exc_off + n_exc * 8;
}

// value j of a 32-value group: its code at bits [K j, K j + K) of w[]
template <int K>
__device__ __forceinline__ uint32_t code_at(const uint32_t* w, int j) {
    const int bit = K * j, wi = bit >> 5, sh = bit & 31;
    uint32_t c = w[wi] >> sh;
    if (sh + K > 32) c |= w[wi + 1] << (32 - sh);
    return c & ((1u << K) - 1u);
}

// one thread per 32-value group: K code words + 32 low bytes in, 64 bytes out
template <int K>
__global__ void __launch_bounds__(256) vcode_decode_kernel(const uint8_t* __restrict__ lo,
                                                           const uint32_t* __restrict__ codes,
                                                           const uint8_t* __restrict__ dict_g, uint64_t nnz,
                                                           uint16_t* __restrict__ out) {
    __shared__ uint32_t dict[128];
    if (threadIdx.x < 128) dict[threadIdx.x] = uint32_t(dict_g[threadIdx.x]) << 8;
    __syncthreads();
    const uint64_t groups = (nnz + 31) / 32;
    for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < groups;
         g += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t w[K + 1];
#pragma unroll
        for (int i = 0; i < K; ++i) w[i] = __ldg(codes + K * g + i);
        w[K] = 0;
        const uint4 l0 = __ldg(reinterpret_cast<const uint4*>(lo + 32 * g));
        const uint4 l1 = __ldg(reinterpret_cast<const uint4*>(lo + 32 * g) + 1);
        const uint32_t lw[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
        uint32_t o[16];
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
            // two values -> one u32 of the output: low bytes spread with PRMT, high bytes from the dictionary
            const uint32_t lb = __byte_perm(lw[j >> 2], 0u, (j & 2) ? 0x4342u : 0x4140u);
            o[j >> 1] = lb | dict[code_at<K>(w, j)] | (dict[code_at<K>(w, j + 1)] << 16);
        }
        uint16_t* dst = out + 32 * g;
        if (32 * g + 32 <= nnz) {
            uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
            for (int q = 0; q < 4; ++q) d4[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        } else {
            const uint32_t rem = uint32_t(nnz - 32 * g);
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (uint32_t(j) < rem) dst[j] = uint16_t(o[j >> 1] >> (16 * (j & 1)));
        }
    }
}

// exceptions: (index << 8) | high byte; indices past nnz are ignored (memory safety)
__global__ void __launch_bounds__(256) vcode_patch_kernel(const unsigned long long* __restrict__ exc, uint64_t n_exc,
                                                          uint64_t nnz, uint16_t* __restrict__ out) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_exc;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const unsigned long long e = exc[i];
        const uint64_t idx = e >> 8;
        if (idx < nnz) out[idx] = uint16_t((out[idx] & 0xFFu) | (uint32_t(e & 0xFFu) << 8));
    }
}

using DecodeFn = void (*)(const uint8_t*, const uint32_t*, const uint8_t*, uint64_t, uint16_t*);
const DecodeFn kDecode[kMaxK + 1] = {nullptr,
                                     vcode_decode_kernel<1>,
                                     vcode_decode_kernel<2>,
                                     vcode_decode_kernel<3>,
                                     vcode_decode_kernel<4>,
                                     vcode_decode_kernel<5>,
                                     vcode_decode_kernel<6>,
                                     vcode_decode_kernel<7>};

// blob header consistent with its own nnz / k / n_exc (offsets recomputed, not trusted)
bool header_ok(const endor_vcode_header* h) {
    if (h->magic != kMagic || h->k < 1 || h->k > uint32_t(kMaxK) || h->n_exc > h->nnz) return false;
    if (h->nnz > (uint64_t(1) << 56)) return false;  // exception entries hold index << 8
    endor_vcode_header e{};
    layout(h->nnz, h->k, h->n_exc, &e);
    return e.lo_off == h->lo_off && e.code_off == h->code_off && e.exc_off == h->exc_off &&
           e.blob_bytes == h->blob_bytes;
}

int nthreads_for(uint64_t nnz) {
    const unsigned hc = std::thread::hardware_concurrency();
    const uint64_t by_size = nnz / (uint64_t(1) << 20) + 1;  // >= 1 Mi values per thread
    return int(std::min<uint64_t>({uint64_t(hc ? hc : 1), 16, by_size}));
}

// run f(t, g0, g1) over [0, groups) split into nt contiguous 32-value group ranges
template <class F>
void parallel_groups(uint64_t groups, int nt, F f) {
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(f, t, groups * t / nt, groups * (t + 1) / nt);
    f(0, 0, groups / nt);
    for (auto& x : th) x.join();
}

}  // namespace

static int values_encode(const void* values_f16, uint64_t nnz, int k_max, void* blob_out, size_t blob_cap,
                         size_t* blob_bytes) {
    if (!blob_bytes) return set_last_error(ENDOR_ERR_INVALID_ARGUMENT, "null blob_bytes");
    if (k_max < 1 || k_max > kMaxK) return set_last_error(ENDOR_ERR_INVALID_ARGUMENT, "k_max must be 1..7");
    if (nnz && !values_f16) return set_last_error(ENDOR_ERR_INVALID_ARGUMENT, "null values");
    if (nnz > (uint64_t(1) << 56)) return set_last_error(ENDOR_ERR_SIZE, "too many values for the exception format");
    const uint8_t* v = static_cast<const uint8_t*>(values_f16);
    const uint64_t groups = (nnz + 31) / 32;
    const int nt = nthreads_for(nnz);
    // 1. histogram of the high bytes
    std::vector<uint64_t> hist_t(size_t(nt) * 256, 0);
    parallel_groups(groups, nt, [&](int t, uint64_t g0, uint64_t g1) {
        uint64_t* hs = &hist_t[size_t(t) * 256];
        const uint64_t e = std::min(nnz, g1 * 32);
        for (uint64_t i = g0 * 32; i < e; ++i) ++hs[v[2 * i + 1]];
    });
    uint64_t hist[256] = {};
    for (int t = 0; t < nt; ++t)
        for (int b = 0; b < 256; ++b) hist[b] += hist_t[size_t(t) * 256 + b];
    // 2. bytes by frequency (ties: smaller byte first, deterministic), best k
    int order[256];
    for (int b = 0; b < 256; ++b) order[b] = b;
    std::stable_sort(order, order + 256, [&](int a, int b) { return hist[a] > hist[b]; });
    endor_vcode_header h{};
    h.magic = kMagic;
    h.nnz = nnz;
    uint64_t best = UINT64_MAX;
    for (uint32_t k = 1; k <= uint32_t(k_max); ++k) {
        uint64_t covered = 0;
        for (uint32_t r = 0; r < (1u << k) - 1u; ++r) covered += hist[order[r]];
        endor_vcode_header c{};
        layout(nnz, k, nnz - covered, &c);
        if (c.blob_bytes < best) {
            best = c.blob_bytes;
            h.k = k;
            h.n_exc = nnz - covered;
        }
    }
    layout(nnz, h.k, h.n_exc, &h);
    *blob_bytes = size_t(h.blob_bytes);
    if (!blob_out) return ENDOR_OK;  // size query
    if (blob_cap < h.blob_bytes) return set_last_error(ENDOR_ERR_INVALID_ARGUMENT, "blob buffer too small");
    const uint32_t k = h.k, esc = (1u << k) - 1u;
    uint8_t code_of[256];
    memset(code_of, uint8_t(esc), sizeof(code_of));
    for (uint32_t r = 0; r < esc; ++r) {
        code_of[order[r]] = uint8_t(r);
        h.dict[r] = uint8_t(order[r]);
    }
    uint8_t* out = static_cast<uint8_t*>(blob_out);
    memcpy(out, &h, sizeof(h));
    uint8_t* lo = out + h.lo_off;
    uint32_t* codes = reinterpret_cast<uint32_t*>(out + h.code_off);
    uint8_t* exc = out + h.exc_off;
    memset(lo + nnz, 0, h.code_off - h.lo_off - nnz);
    memset(reinterpret_cast<uint8_t*>(codes) + groups * k * 4, 0, h.exc_off - h.code_off - groups * k * 4);
    // 3. low bytes, packed codes, and each thread's exceptions (concatenated in index order)
    std::vector<std::vector<unsigned long long>> ex_t(nt);
    parallel_groups(groups, nt, [&](int t, uint64_t g0, uint64_t g1) {
        auto& ex = ex_t[t];
        for (uint64_t g = g0; g < g1; ++g) {
            uint32_t w[kMaxK + 1] = {};
            const uint64_t e = std::min<uint64_t>(32, nnz - 32 * g);
            for (uint64_t j = 0; j < e; ++j) {
                const uint64_t i = 32 * g + j;
                const uint8_t hi = v[2 * i + 1];
                lo[i] = v[2 * i];
                const uint32_t c = code_of[hi];
                if (c == esc) ex.push_back((static_cast<unsigned long long>(i) << 8) | hi);
                const uint32_t bit = k * uint32_t(j), wi = bit >> 5, sh = bit & 31;
                w[wi] |= c << sh;
                if (sh + k > 32) w[wi + 1] |= c >> (32 - sh);
            }
            memcpy(codes + g * k, w, k * 4);
        }
    });
    for (auto& ex : ex_t) {
        memcpy(exc, ex.data(), ex.size() * 8);
        exc += ex.size() * 8;
    }
    return ENDOR_OK;
}

extern "C" {

int endor_values_encode(const void* values_f16, uint64_t nnz, int k_max, void* blob_out, size_t blob_cap,
                        size_t* blob_bytes) {
    try {  // worker threads and buffers: no C++ exception crosses the C ABI
        return values_encode(values_f16, nnz, k_max, blob_out, blob_cap, blob_bytes);
    } catch (const std::exception& e) {
        return set_last_error(ENDOR_ERR_CUDA, (std::string("host encoder: ") + e.what()).c_str());
    }
}

int endor_values_decode_host_check(const void* header_host) {
    if (!header_host) return set_last_error(ENDOR_ERR_INVALID_ARGUMENT, "null header");
    if (!header_ok(static_cast<const endor_vcode_header*>(header_host)))
        return set_last_error(ENDOR_ERR_CORRUPTION, "coded-values header is inconsistent");
    return ENDOR_OK;
}

int endor_cuda_values_decode(const void* header_host, const void* blob_dev, void* values_out, void* stream) {
    int st;
    if ((st = endor_values_decode_host_check(header_host))) return st;
    const auto* h = static_cast<const endor_vcode_header*>(header_host);
    if (h->nnz == 0) return ENDOR_OK;
    if (!blob_dev || !values_out || reinterpret_cast<uintptr_t>(blob_dev) % 16 ||
        reinterpret_cast<uintptr_t>(values_out) % 16)
        return set_last_error(ENDOR_ERR_INVALID_ARGUMENT, "blob and output must be non-null and 16-byte aligned");
    const uint8_t* b = static_cast<const uint8_t*>(blob_dev);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t groups = (h->nnz + 31) / 32;
    const unsigned grid = unsigned(std::min<uint64_t>((groups + 255) / 256, uint64_t(sms) * 8));
    kDecode[h->k]<<<grid, 256, 0, s>>>(b + h->lo_off, reinterpret_cast<const uint32_t*>(b + h->code_off),
                                       b + offsetof(endor_vcode_header, dict), h->nnz,
                                       static_cast<uint16_t*>(values_out));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_last_error(ENDOR_ERR_CUDA, cudaGetErrorString(e));
    if (h->n_exc) {
        const unsigned pg = unsigned(std::min<uint64_t>((h->n_exc + 255) / 256, uint64_t(sms) * 8));
        vcode_patch_kernel<<<pg, 256, 0, s>>>(reinterpret_cast<const unsigned long long*>(b + h->exc_off), h->n_exc,
                                              h->nnz, static_cast<uint16_t*>(values_out));
        e = cudaGetLastError();
        if (e != cudaSuccess) return set_last_error(ENDOR_ERR_CUDA, cudaGetErrorString(e));
    }
    return ENDOR_OK;
}

}  // extern "C"
