// common.cuh -- shared constants, workspace layout and device helpers for the
// sm_100a Endor decompression path.  See DESIGN.md for the data layout.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "endor_cuda.h"

namespace endor_b200 {

// ---- geometry --------------------------------------------------------------
// Expand tile: 8192 elements per CTA pass (= 256 u32 bitmap words, one per
// thread).  A power of two, so every RankIndex chunk size <= it divides it.
constexpr int kTileElems = 8192;
constexpr int kTileWords = kTileElems / 32;  // 256
constexpr int kExpandThreads = 256;

// Scan (rank) kernel: 8 warps x 16 iterations x 32 lanes of u32 words.
constexpr int kScanThreads = 256;
constexpr int kScanWordsPerLane = 16;
constexpr int kScanWarpWords = 32 * kScanWordsPerLane;                   // 512
constexpr int kScanBlockWords = (kScanThreads / 32) * kScanWarpWords;    // 4096
constexpr uint64_t kScanBlockBits = uint64_t(kScanBlockWords) * 32;     // 131072

// count_kernel (hot path): count blocks of kCountBlockWords u32 words
// (16 KiB = 128 sub-tiles of 1024 bits), streamed through a kCountStages-deep
// TMA ring per CTA (3 blocks in flight while one is counted).
#ifndef ENDOR_COUNT_BLOCK_WORDS
#define ENDOR_COUNT_BLOCK_WORDS 4096
#endif
#ifndef ENDOR_COUNT_STAGES
#define ENDOR_COUNT_STAGES 4
#endif
constexpr int kCountBlockWords = ENDOR_COUNT_BLOCK_WORDS;
constexpr int kCountSubs = kCountBlockWords / 32;  // sub-tiles per count block
constexpr int kCountStages = ENDOR_COUNT_STAGES;

// ---- workspace ---------------------------------------------------------------
// [0,256)                 WsHeader
// [256, +8*(ntiles+1))    per-tile exclusive value offsets ("GPU RankIndex")
// [.., +8*nscan)          decoupled look-back state of the scan kernel
// [.., +8*32768)          magnitude_prune key histogram
// [.., +8*(ntiles+1))     magnitude_prune per-tile tie counts / prefixes
struct WsHeader {
    uint32_t status;       // latched endor_status (0 = OK)
    uint32_t pad0;
    unsigned long long ticket;  // scan CTA ticket counter (self-resetting)
    unsigned long long done;    // scan CTA completion counter (self-resetting)
    unsigned long long total;   // last scan total (p0 + popcount of range)
    unsigned long long aux[4];
    unsigned long long tile_claim;  // expand_tma_kernel's global tile-claim counter (self-resetting)
    unsigned long long tile_done;   // ... and its count of claimers done (self-resetting)
};
static_assert(sizeof(WsHeader) <= 256, "the workspace header occupies the first 256 bytes");

struct WsLayout {
    WsHeader* hdr;
    unsigned long long* tprefix;
    unsigned long long* lookback;
    unsigned long long* hist;
    unsigned long long* ties;
    unsigned long long* tsub;  // per-1024-element sub-tile value offsets
    unsigned long long* blk;   // count_kernel per-CTA bases (+ total)
    float* part;               // fused GEMV: one fp32 partial per sub-tile
    uint64_t ntiles, nscan, nsub;
    size_t bytes;
};

constexpr int kSubElems = 1024;  // granularity of the value-offset tables (count_kernel / RankIndex)

// Expand consumers per TMA-kernel CTA: each handles kWarpElems elements of a
// tile.  8 x 1024 measured 0.893 of roofline vs 0.678 for 16 x 512
// (profiles/r01/README.md): per-warp ILP beats more, thinner warps here.
#ifndef ENDOR_CONSUMER_WARPS
#define ENDOR_CONSUMER_WARPS 8
#endif
constexpr int kConsumerWarps = ENDOR_CONSUMER_WARPS;
constexpr int kWarpElems = kTileElems / kConsumerWarps;  // 512 (or 1024 with 8 warps)
constexpr int kWarpWords = kWarpElems / 32;

__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// n sizes the per-tensor regions; sub_cap / blk_cap size the count_kernel
// arrays (a batch of tensors needs the sum of theirs, see batch_plan).
inline WsLayout ws_layout_caps(void* base, uint64_t n, uint64_t sub_cap, uint64_t blk_cap) {
    WsLayout L{};
    L.ntiles = ceil_div(n, kTileElems);
    L.nscan = ceil_div(n, kScanBlockBits);
    L.nsub = ceil_div(n, kSubElems);
    size_t off = 256;
    char* b = static_cast<char*>(base);
    L.hdr = reinterpret_cast<WsHeader*>(b);
    L.tsub = reinterpret_cast<unsigned long long*>(b + off);
    off = align256(off + 8 * sub_cap);
    L.blk = reinterpret_cast<unsigned long long*>(b + off);
    off = align256(off + 8 * blk_cap);
    L.part = reinterpret_cast<float*>(b + off);  // fused-GEMV partials, one per consumer warp-tile
    off = align256(off + 4 * sub_cap * (kSubElems / kWarpElems));
    L.tprefix = reinterpret_cast<unsigned long long*>(b + off);
    off = align256(off + 8 * (L.ntiles + 1));
    L.lookback = reinterpret_cast<unsigned long long*>(b + off);  // must stay zeroed between calls
    off = align256(off + 8 * (L.nscan + 1));
    L.hist = reinterpret_cast<unsigned long long*>(b + off);
    off = align256(off + 8 * 32768);
    L.ties = reinterpret_cast<unsigned long long*>(b + off);
    off = align256(off + 8 * (L.ntiles + 1));
    L.bytes = off;
    return L;
}

inline WsLayout ws_layout(void* base, uint64_t n) {
    return ws_layout_caps(base, n, (ceil_div(n, kSubElems) + 16 + 7) & ~uint64_t(7),
                          ceil_div(n, kScanBlockBits) + 2);
}

// ---- f16 bit math, float16.hpp:35-73 (device restatement) -------------------
__device__ __forceinline__ uint16_t f32_to_f16_bits(float f) {
    const uint32_t x = __float_as_uint(f);
    const uint16_t sign = uint16_t((x >> 16) & 0x8000u);
    const uint32_t mag = x & 0x7FFFFFFFu;
    if (mag >= 0x7F800000u) {
        if (mag == 0x7F800000u) return uint16_t(sign | 0x7C00u);
        uint16_t payload = uint16_t((mag >> 13) & 0x3FFu);
        if (payload == 0) payload = 0x200u;
        return uint16_t(sign | 0x7C00u | payload);
    }
    if (mag >= 0x477FF000u) return uint16_t(sign | 0x7C00u);
    const uint32_t exp = mag >> 23;
    if (exp >= 0x71u) {
        const uint32_t mant = mag & 0x7FFFFFu;
        uint32_t half = ((exp - 0x70u) << 10) | (mant >> 13);
        const uint32_t rem = mant & 0x1FFFu;
        half += (rem > 0x1000u) || (rem == 0x1000u && (half & 1u));
        return uint16_t(sign | half);
    }
    const uint32_t m24 = (mag & 0x7FFFFFu) | 0x800000u;
    const uint32_t shift = 126u - exp;
    if (shift > 24u) return sign;
    uint32_t m = m24 >> shift;
    const uint32_t rem = m24 & ((1u << shift) - 1u);
    const uint32_t halfway = 1u << (shift - 1);
    m += (rem > halfway) || (rem == halfway && (m & 1u));
    return uint16_t(sign | m);
}

// ---- PTX wrappers: shared memory, mbarrier, TMA bulk copies -------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ unsigned long long lds64(uint32_t addr) {
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts8(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(bar), "r"(parity) : "memory");
}
// Orders this thread's generic-proxy shared-memory writes before later
// async-proxy (TMA) accesses of the same bytes: the producers patch buffer
// edges with st.shared into stage buffers a later cp.async.bulk overwrites.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on an mbarrier.
// dst/src 16-byte aligned, bytes a multiple of 16.
#ifndef ENDOR_BULK_EVICT_FIRST
#define ENDOR_BULK_EVICT_FIRST 0
#endif
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
#if ENDOR_BULK_EVICT_FIRST
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory");
#else
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
#endif
}

// ---- programmatic dependent launch (PDL) ------------------------------------------
// The hot-path kernels (count -> expand / fused GEMV -> row sum) are launched
// with cudaLaunchAttributeProgrammaticStreamSerialization: a dependent grid's
// CTAs start (launch latency, mbarrier / LUT prologue) while the previous
// kernel drains, and block in pdl_wait() -- which returns once the previous
// grid has completed and its memory is visible -- before reading anything it
// produced (workspace tables, the latched status).  Without the attribute both
// are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- device helpers ------------------------------------------------------------
// Little-endian u32 bitmap word `w`; bytes at or past `nbytes` read as zero
// (only the final word of a bitmap can be partial).
__device__ __forceinline__ uint32_t load_word32(const uint8_t* __restrict__ bm, uint64_t w,
                                                uint64_t nbytes) {
    const uint64_t b0 = w * 4;
    if (b0 + 4 <= nbytes) return __ldg(reinterpret_cast<const uint32_t*>(bm) + w);
    uint32_t v = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (b0 + j < nbytes) v |= uint32_t(__ldg(bm + b0 + j)) << (8 * j);
    return v;
}

__device__ __forceinline__ void latch_status(WsHeader* hdr, uint32_t code) {
    atomicCAS(&hdr->status, 0u, code);
}

__device__ __forceinline__ uint32_t read_status(const WsHeader* hdr) {
    return *reinterpret_cast<const volatile uint32_t*>(&hdr->status);
}

// CTA-uniform view of the latched status: thread 0 reads it once and one
// barrier broadcasts the answer, so a latch landing mid-read can never split
// a CTA (warp-specialised kernels would otherwise leave a producer or its
// consumers waiting on an mbarrier forever).  Call from every thread.
__device__ __forceinline__ bool cta_error_latched(const WsHeader* hdr) {
    return __syncthreads_or(threadIdx.x == 0 && read_status(hdr) != 0) != 0;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += u;
    }
    return v;
}

// Exclusive warp prefix sum of small values (0..63) by bit-slicing: six
// independent ballots instead of a five-deep dependent shuffle chain.
__device__ __forceinline__ uint32_t warp_excl_scan_small(uint32_t v) {
    uint32_t lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    uint32_t r = 0;
#pragma unroll
    for (int b = 0; b < 6; ++b) r += uint32_t(__popc(__ballot_sync(0xffffffffu, (v >> b) & 1u) & lt)) << b;
    return r;
}

// Look-back state word: [63:62] flag (1 = aggregate, 2 = inclusive prefix),
// [61:0] value.
constexpr unsigned long long kLbAgg = 1ull << 62;
constexpr unsigned long long kLbPrefix = 2ull << 62;
constexpr unsigned long long kLbValue = (1ull << 62) - 1;

__device__ __forceinline__ void lb_store(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

}  // namespace endor_b200
