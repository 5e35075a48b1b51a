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
#include <queue>
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

// ---- Huffman mode ("EVH1"): the high bytes as a canonical Huffman stream, in
// chunks of 512 values that each start on a 32-bit word (offsets table), so a
// thread decodes a chunk on its own through a 4096-entry lookup table
// (symbol | length << 8, indexed by the next 12 stream bits, LSB first)
// shipped in the blob.  Layout: header | LUT (8 KiB) | lo (nnz, padded to 32)
// | chunk word offsets (u32 x (chunks + 1), padded to 16) | stream (u32
// words, zero-padded to 16 bytes; header n_exc = their count).
constexpr uint32_t kMagicH = 0x31485645u;  // "EVH1"
constexpr int kHuffBits = 12;              // longest code = LUT index width
constexpr uint64_t kHuffChunk = 512;

void layout_huff(uint64_t nnz, uint64_t words, endor_vcode_header* h) {
    h->lo_off = sizeof(endor_vcode_header) + (uint64_t(2) << kHuffBits);
    h->code_off = h->lo_off + up(nnz, 32);
    h->exc_off = h->code_off + up(((nnz + kHuffChunk - 1) / kHuffChunk + 1) * 4, 16);
    h->blob_bytes = h->exc_off + up(words * 4, 16);  // whole 16-byte blocks (the decoder's loads)
}

// CTA = 128 threads = 128 consecutive chunks, whose streams are contiguous:
// the CTA stages that word range in shared memory with coalesced loads, then
// each thread decodes its chunk from there (a shared-memory refill every ~10
// symbols instead of a dependent global load) and writes 4 values per step.
// A range larger than the buffer (high-entropy high bytes) is read from
// global memory instead: same result, slower.
constexpr int kHuffThreads = 128;
constexpr uint32_t kHuffStageWords = 12288;  // 48 KiB: up to 6 bits per value on average
constexpr uint32_t kHuffSmem = (2u << kHuffBits) + kHuffStageWords * 4;

__global__ void __launch_bounds__(kHuffThreads) vcode_huff_kernel(const uint16_t* __restrict__ lut_g,
                                                                  const uint8_t* __restrict__ lo,
                                                                  const uint32_t* __restrict__ offs,
                                                                  const uint32_t* __restrict__ stream,
                                                                  uint64_t words, uint64_t nnz,
                                                                  uint16_t* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t sm[];
    uint16_t* lut = reinterpret_cast<uint16_t*>(sm);
    uint32_t* sw = reinterpret_cast<uint32_t*>(sm + (2u << kHuffBits));
    const int tid = threadIdx.x;
    for (int i = tid; i < (1 << kHuffBits) / 2; i += kHuffThreads)
        reinterpret_cast<uint32_t*>(lut)[i] = __ldg(reinterpret_cast<const uint32_t*>(lut_g) + i);
    const uint64_t chunks = (nnz + kHuffChunk - 1) / kHuffChunk;
    for (uint64_t blk = blockIdx.x; blk * kHuffThreads < chunks; blk += gridDim.x) {
        const uint64_t c0 = blk * kHuffThreads, c1 = umin64(c0 + kHuffThreads, chunks);
        // the CTA's word range (a corrupt offsets table cannot move reads outside the stream)
        const uint64_t w0 = umin64(offs[c0], words), w1 = umin64(umin64(offs[c1], words), w0 + (uint64_t(1) << 31));
        const bool staged = w1 - w0 <= kHuffStageWords;
        __syncthreads();  // the previous step's reads of sw are done
        if (staged)
            for (uint32_t i = tid; i < uint32_t(w1 - w0); i += kHuffThreads) sw[i] = __ldg(stream + w0 + i);
        __syncthreads();
        const uint64_t c = c0 + tid;
        if (c >= c1) continue;
        const uint64_t e = umin64(offs[c + 1], words), b = umin64(offs[c], e);
        const uint32_t* src = staged ? sw : stream + w0;
        uint32_t p = uint32_t(umin64(b, w1) - w0), pend = uint32_t(umin64(e, w1) - w0);
        uint64_t buf = 0;
        uint32_t nb = 0;
        const uint64_t v0 = c * kHuffChunk;
        const uint32_t cnt = uint32_t(umin64(kHuffChunk, nnz - v0));
        // low bytes 16 at a time, the next 16 loaded one block (16 symbols) ahead
        const uint4* lo4 = reinterpret_cast<const uint4*>(lo + v0);
        uint4 cur = __ldg(lo4);
        for (uint32_t j = 0; j < cnt; j += 16) {
            const uint4 nxt = j + 16 < cnt ? __ldg(lo4 + j / 16 + 1) : make_uint4(0, 0, 0, 0);
            const uint32_t lw[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
            for (int s4 = 0; s4 < 4; ++s4) {
                const uint32_t jj = j + 4 * s4;
                if (jj >= cnt) break;
                uint32_t hi4 = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (nb < uint32_t(kHuffBits)) {
                        buf |= uint64_t(p < pend ? src[p] : 0u) << nb;
                        ++p;
                        nb += 32;
                    }
                    const uint32_t en = lut[buf & ((1u << kHuffBits) - 1u)], len = en >> 8;
                    buf >>= len;
                    nb -= len;
                    hi4 |= (en & 0xFFu) << (8 * q);
                }
                const uint2 o = make_uint2(__byte_perm(lw[s4], hi4, 0x5140), __byte_perm(lw[s4], hi4, 0x7362));
                if (jj + 4 <= cnt) {
                    *reinterpret_cast<uint2*>(out + v0 + jj) = o;
                } else {
                    for (uint32_t q = 0; q < cnt - jj; ++q)
                        out[v0 + jj + q] = uint16_t((q < 2 ? o.x : o.y) >> (16 * (q & 1)));
                }
            }
            cur = nxt;
        }
    }
}

// Huffman code lengths <= kHuffBits (frequencies flattened until they fit)
void huff_lengths(const uint64_t* hist, uint8_t* len) {
    std::vector<uint64_t> f(hist, hist + 256);
    for (;;) {
        struct Node { uint64_t w; int l, r; };  // leaf: l = -1, r = symbol
        std::vector<Node> nodes;
        using P = std::pair<uint64_t, int>;
        std::priority_queue<P, std::vector<P>, std::greater<P>> pq;
        for (int s = 0; s < 256; ++s)
            if (f[s]) {
                nodes.push_back({f[s], -1, s});
                pq.push({f[s], int(nodes.size()) - 1});
            }
        memset(len, 0, 256);
        if (nodes.empty()) return;
        if (nodes.size() == 1) {
            len[nodes[0].r] = 1;
            return;
        }
        while (pq.size() > 1) {
            const P a = pq.top();
            pq.pop();
            const P b = pq.top();
            pq.pop();
            nodes.push_back({a.first + b.first, a.second, b.second});
            pq.push({a.first + b.first, int(nodes.size()) - 1});
        }
        int maxd = 0;
        std::vector<std::pair<int, int>> st{{int(nodes.size()) - 1, 0}};
        while (!st.empty()) {
            const auto [n, d] = st.back();
            st.pop_back();
            if (nodes[n].l < 0) {
                len[nodes[n].r] = uint8_t(d);
                maxd = std::max(maxd, d);
            } else {
                st.push_back({nodes[n].l, d + 1});
                st.push_back({nodes[n].r, d + 1});
            }
        }
        if (maxd <= kHuffBits) return;
        for (auto& x : f)
            if (x) x = (x >> 1) | 1;
    }
}

// canonical codes (first bit at bit 0 of the stream), and the decode table
void huff_codes(const uint8_t* len, uint32_t* rev, uint16_t* lut) {
    uint32_t code = 0;
    for (int L = 1; L <= kHuffBits; ++L) {
        for (int s = 0; s < 256; ++s)
            if (len[s] == L) {
                uint32_t r = 0;
                for (int b = 0; b < L; ++b) r |= ((code >> b) & 1u) << (L - 1 - b);
                rev[s] = r;
                ++code;
            }
        code <<= 1;
    }
    for (int s = 0; s < 256; ++s)
        if (len[s])
            for (uint32_t h = 0; h < (1u << (kHuffBits - len[s])); ++h)
                lut[rev[s] | (h << len[s])] = uint16_t(s | (len[s] << 8));
}

// blob header consistent with its own nnz / k / n_exc (offsets recomputed, not trusted)
bool header_ok(const endor_vcode_header* h) {
    if (h->magic == kMagicH) {
        if (h->k != uint32_t(kHuffBits) || h->nnz > (uint64_t(1) << 40) || h->n_exc > (uint64_t(1) << 32)) return false;
        endor_vcode_header e{};
        layout_huff(h->nnz, h->n_exc, &e);
        return e.lo_off == h->lo_off && e.code_off == h->code_off && e.exc_off == h->exc_off &&
               e.blob_bytes == h->blob_bytes;
    }
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
    if (k_max < 0 || k_max > kMaxK)
        return set_last_error(ENDOR_ERR_INVALID_ARGUMENT, "k_max must be 0 (automatic) or 1..7");
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
    for (uint32_t k = 1; k <= uint32_t(k_max ? k_max : kMaxK); ++k) {
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
    if (k_max == 0 && nnz > 0 && nnz <= (uint64_t(1) << 40)) {
        // automatic: the Huffman stream when it is smaller (exact size: per-chunk word counts)
        uint8_t len[256];
        huff_lengths(hist, len);
        const uint64_t chunks = (nnz + kHuffChunk - 1) / kHuffChunk;
        std::vector<uint32_t> cw(chunks + 1, 0);
        parallel_groups(chunks, nt, [&](int, uint64_t c0, uint64_t c1) {
            for (uint64_t c = c0; c < c1; ++c) {
                uint64_t bits = 0;
                const uint64_t e = std::min(nnz, (c + 1) * kHuffChunk);
                for (uint64_t i = c * kHuffChunk; i < e; ++i) bits += len[v[2 * i + 1]];
                cw[c] = uint32_t((bits + 31) / 32);
            }
        });
        uint64_t words = 0;
        for (uint64_t c = 0; c < chunks; ++c) {
            const uint32_t w = cw[c];
            cw[c] = uint32_t(words);  // exclusive prefix: the chunk's first word
            words += w;
        }
        cw[chunks] = uint32_t(words);
        endor_vcode_header hh{};
        layout_huff(nnz, words, &hh);
        if (words < (uint64_t(1) << 32) && hh.blob_bytes < h.blob_bytes) {
            hh.magic = kMagicH;
            hh.k = kHuffBits;
            hh.nnz = nnz;
            hh.n_exc = words;
            *blob_bytes = size_t(hh.blob_bytes);
            if (!blob_out) return ENDOR_OK;  // size query
            if (blob_cap < hh.blob_bytes) return set_last_error(ENDOR_ERR_INVALID_ARGUMENT, "blob buffer too small");
            uint32_t rev[256] = {};
            uint8_t* out = static_cast<uint8_t*>(blob_out);
            memcpy(out, &hh, sizeof(hh));
            memset(out + sizeof(hh), 0, hh.lo_off - sizeof(hh));
            huff_codes(len, rev, reinterpret_cast<uint16_t*>(out + sizeof(hh)));
            uint8_t* lo = out + hh.lo_off;
            memset(lo + nnz, 0, hh.code_off - hh.lo_off - nnz);
            memset(out + hh.code_off, 0, hh.exc_off - hh.code_off);
            memcpy(out + hh.code_off, cw.data(), (chunks + 1) * 4);
            uint32_t* stream = reinterpret_cast<uint32_t*>(out + hh.exc_off);
            memset(stream + words, 0, hh.blob_bytes - hh.exc_off - words * 4);
            parallel_groups(chunks, nt, [&](int, uint64_t c0, uint64_t c1) {
                for (uint64_t c = c0; c < c1; ++c) {
                    uint32_t* wp = stream + cw[c];
                    uint64_t acc = 0;
                    uint32_t nb = 0;
                    const uint64_t e = std::min(nnz, (c + 1) * kHuffChunk);
                    for (uint64_t i = c * kHuffChunk; i < e; ++i) {
                        const uint8_t hi = v[2 * i + 1];
                        lo[i] = v[2 * i];
                        acc |= uint64_t(rev[hi]) << nb;
                        nb += len[hi];
                        if (nb >= 32) {
                            *wp++ = uint32_t(acc);
                            acc >>= 32;
                            nb -= 32;
                        }
                    }
                    if (nb) *wp = uint32_t(acc);
                }
            });
            return ENDOR_OK;
        }
    }
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
    if (h->magic == kMagicH) {
        const uint64_t chunks = (h->nnz + kHuffChunk - 1) / kHuffChunk;
        const cudaError_t attr = cudaFuncSetAttribute(
            vcode_huff_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kHuffSmem));
        if (attr != cudaSuccess) return set_last_error(ENDOR_ERR_CUDA, cudaGetErrorString(attr));
        const unsigned hg = unsigned(std::min<uint64_t>((chunks + kHuffThreads - 1) / kHuffThreads, uint64_t(sms) * 4));
        vcode_huff_kernel<<<hg, kHuffThreads, kHuffSmem, s>>>(reinterpret_cast<const uint16_t*>(b + sizeof(endor_vcode_header)),
                                             b + h->lo_off, reinterpret_cast<const uint32_t*>(b + h->code_off),
                                             reinterpret_cast<const uint32_t*>(b + h->exc_off), h->n_exc, h->nnz,
                                             static_cast<uint16_t*>(values_out));
        cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? ENDOR_OK : set_last_error(ENDOR_ERR_CUDA, cudaGetErrorString(e));
    }
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
