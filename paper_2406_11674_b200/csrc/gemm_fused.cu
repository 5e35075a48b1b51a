// gemm_fused.cu -- fused decompress -> GEMM on the 5th-generation tensor cores.
//
// Y[t, r] = sum_c W[r, c] X[t, c] for an offloaded layer's W held in the
// Endor format (bitmap + packed f16 values, codec.hpp:24-66), i.e. the
// prefill / batched-decode consumer of the decompressed weights (north star
// (b) "dense GEMV/GEMM consumer"; the reference only models the consumer as a
// constant, sim.hpp:30,256).  The dense W is never written to HBM: each CTA
// expands its W tile straight into shared memory in the UMMA canonical layout
// and feeds it to tcgen05.mma as the A operand.
//
// Tile: 128 W rows (UMMA M) x BN tokens (UMMA N) x the CTA's K range, fp32
// accumulator in TMEM (BN columns).  Per CTA (384 threads, 1 per SM):
//   warps 0, 3  raw producers (64 rows each): per 128-column span, the span's
//               bitmap (16 bytes per row, cp.async a few spans ahead) and every
//               row's packed-values window (16-byte aligned superset, copied
//               by 8 lanes per row with 16-byte cp.async) into a raw ring; row
//               value cursors advance by popc.  (One 1-D bulk copy per row
//               window -- 128 per span -- was TMA-issue-bound: 0.08 of roofline.)
//   warp 1      X producer: 2-D TMA (128-byte swizzle) of each 64-column
//               k-block's BN x 64 X tile
//   warp 2      TMEM allocator + MMA issuer (one elected lane): 4 x
//               tcgen05.mma.kind::f16 (K = 16) per k-block, commit -> empty
//   warps 4-11  expand: thread = (row, half of the k-block's 8 chunks); the
//               selector/PRMT gather of gather.cuh writes 16-byte chunks into
//               the A stage at the 128-byte-swizzle position; fence.proxy.async
//               + mbarrier arrive hands the stage to the MMA.  After the K loop
//               the same warps drain TMEM (tcgen05.ld 32x32b) and write Y (or a
//               split-K fp32 partial) with coalesced stores.
// Row starts come from a flat 1024-element RankIndex (the caller's prefix1024
// or count_kernel + flatten) plus the popcount of the bits since the chunk
// start; every row's final cursor is checked against the rank of its range
// end (= nnz for the last row: check_index, codec.hpp:170-184), and every
// copy is clamped to the values buffer, so an inconsistent index latches
// CorruptionError and never reads outside the inputs.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "gather.cuh"
#include "kernels.h"

// development switch (tools/build_variant.sh): bit 0 no MMA, bit 1 no gather
// (A left stale), bit 2 no value copies -- isolates the pipeline's limiter
#ifndef ENDOR_GEMM_SKIP
#define ENDOR_GEMM_SKIP 0
#endif

namespace endor_b200 {

constexpr int kGmRows = 128;                        // UMMA M
constexpr int kGmKB = 64;                           // k-block: 64 f16 = one 128-byte swizzle row
constexpr int kGmSpan = 128;                        // bitmap span: 2 k-blocks, 16 bytes per row
constexpr int kGmWin = 80;                          // per-thread values window: <= 32 values + 16-byte slack
constexpr int kGmExpandWarps = 16;
constexpr int kGmExpandThreads = kGmExpandWarps * 32;
constexpr int kGmRawBytes = kGmExpandThreads * kGmWin;  // one span's windows: 40 KiB
constexpr int kGmBmpBytes = kGmRows * 16;           // 2048
constexpr int kGmThreads = (4 + kGmExpandWarps) * 32;  // 640
constexpr int kGmBmp = 8;                           // bitmap ring (spans)

constexpr int kGmAS = 8;                           // A stages, in TMEM (32 columns each)

template <int BN>
struct GmCfg {
    static constexpr int kXS = BN == 64 ? 8 : (BN == 128 ? 5 : 3);  // X stages (TMA ring in smem)
    static constexpr int kLook = BN == 256 ? 1 : 2;                 // spans of value copies in flight per thread
    static constexpr int kRaw = kLook + 1;                          // private window slots per thread
    static constexpr uint32_t kTmemCols = BN + 32 * kGmAS <= 256 ? 256 : 512;  // accumulator + A stages
    static constexpr uint32_t kB = 0;                             // X tiles, BN x 128 bytes (1024-aligned)
    static constexpr uint32_t kRawOff = kB + kXS * BN * 128;
    static constexpr uint32_t kBmpOff = kRawOff + kRaw * kGmRawBytes;
    static constexpr uint32_t kBar = kBmpOff + kGmBmp * kGmBmpBytes;
    // xfull[kXS] xempty[kXS] afull[kAS] aempty[kAS] bmp_full[kBmp] bmp_empty[kBmp] tmem_full, tmem addr
    static constexpr uint32_t kTmemSlot = kBar + 8 * (2 * kXS + 2 * kGmAS + 2 * kGmBmp + 1);
    static constexpr uint32_t kRank = (kTmemSlot + 4 + 15) & ~15u;  // u64 start[128], end[128]
    static constexpr uint32_t kEnd = kRank + 2 * 8 * kGmRows + 16;  // + gather over-read pad
    static constexpr uint32_t kSmem = kEnd + 1024;                  // + alignment of the dynamic base
};
static_assert(GmCfg<256>::kSmem + 1024 <= 232448 && GmCfg<128>::kSmem + 1024 <= 232448 &&
                  GmCfg<64>::kSmem + 1024 <= 232448,
              "GEMM shared-memory plan exceeds 227 KiB (incl. 1 KiB static)");

struct GemmArgs {
    const uint8_t* bitmap;
    uint64_t nbytes;
    const uint8_t* values;
    uint64_t nnz;
    const unsigned long long* idx;  // flat RankIndex at chunk 1024 (absolute offsets)
    uint64_t rows, cols, tokens;
    uint32_t m_tiles, n_tiles, ksplit, sps;  // sps: 128-column spans per split
    uint64_t nspans;                         // spans per row: ceil(cols / 128)
    float* part;                             // ksplit > 1: [ksplit][tokens][rows]
    float* y32;                              // ksplit == 1
    __half* y16;
    WsHeader* hdr;
    int bmp_async;                           // cols % 128 == 0 and 16-byte aligned bitmap: cp.async rows
};

// ---- tcgen05 / TMA wrappers -------------------------------------------------------
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar) : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
// K-major operand, 128-byte swizzle: rows of 128 bytes, 8-row groups 1024 bytes apart
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
           (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
}
// A from TMEM (lane = M row, K elements packed 2 per 32-bit column), B from shared memory
__device__ __forceinline__ void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bd, uint32_t idesc,
                                            uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(tmem_d), "r"(tmem_a), "l"(bd), "r"(idesc), "r"(acc) : "memory");
}
// this warp's 32 TMEM lanes, 32 consecutive 32-bit columns from 8 x uint4 per thread
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint4 (&v)[8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
        ::"r"(taddr), "r"(v[0].x), "r"(v[0].y), "r"(v[0].z), "r"(v[0].w), "r"(v[1].x), "r"(v[1].y), "r"(v[1].z),
          "r"(v[1].w), "r"(v[2].x), "r"(v[2].y), "r"(v[2].z), "r"(v[2].w), "r"(v[3].x), "r"(v[3].y), "r"(v[3].z),
          "r"(v[3].w), "r"(v[4].x), "r"(v[4].y), "r"(v[4].z), "r"(v[4].w), "r"(v[5].x), "r"(v[5].y), "r"(v[5].z),
          "r"(v[5].w), "r"(v[6].x), "r"(v[6].y), "r"(v[6].z), "r"(v[6].w), "r"(v[7].x), "r"(v[7].y), "r"(v[7].z),
          "r"(v[7].w)
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint4 (&v)[4]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(taddr), "r"(v[0].x), "r"(v[0].y), "r"(v[0].z), "r"(v[0].w), "r"(v[1].x), "r"(v[1].y), "r"(v[1].z),
          "r"(v[1].w), "r"(v[2].x), "r"(v[2].y), "r"(v[2].z), "r"(v[2].w), "r"(v[3].x), "r"(v[3].y), "r"(v[3].z),
          "r"(v[3].w)
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

// rank(p) for p < n from the flat 1024-element table plus the popcount of
// the bits [1024 (p / 1024), p); one warp, result in every lane
__device__ __forceinline__ unsigned long long warp_rank(const GemmArgs& a, uint64_t p, int lane) {
    const uint64_t j = p >> 10;
    const uint32_t rem = uint32_t(p & 1023u);
    const uint64_t w = (j << 5) + lane;
    uint32_t v = 0;
    if (uint32_t(lane) * 32 < rem) {
        v = load_word32(a.bitmap, w, a.nbytes);
        const uint32_t valid = rem - uint32_t(lane) * 32;
        if (valid < 32) v &= (1u << valid) - 1u;
    }
    const uint32_t pc = __reduce_add_sync(0xffffffffu, uint32_t(__popc(v)));
    return __ldg(a.idx + j) + pc;
}

template <int BN>
__global__ void __launch_bounds__(kGmThreads, 1)
    gemm_fused_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ GemmArgs a) {
    using C = GmCfg<BN>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t sraw = smem_u32(smem_raw);
    const uint32_t sb = (sraw + 1023u) & ~1023u;  // swizzle-128B operands need 1024-byte alignment
    uint8_t* const smem = smem_raw + (sb - sraw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    const uint32_t xfull0 = sb + C::kBar, xempty0 = xfull0 + 8 * C::kXS;
    const uint32_t afull0 = xempty0 + 8 * C::kXS, aempty0 = afull0 + 8 * kGmAS;
    const uint32_t bfull0 = aempty0 + 8 * kGmAS, bempty0 = bfull0 + 8 * kGmBmp, tfull = bempty0 + 8 * kGmBmp;
    unsigned long long* const rstart = reinterpret_cast<unsigned long long*>(smem + C::kRank);
    unsigned long long* const rend = rstart + kGmRows;

    // work unit: n-tile fastest, so the CTAs sharing a W tile run together (L2 reuse)
    uint32_t u = blockIdx.x;
    const uint32_t nt = u % a.n_tiles;
    u /= a.n_tiles;
    const uint32_t ks = u % a.ksplit, mt = u / a.ksplit;
    const uint64_t m0 = uint64_t(mt) * kGmRows;
    const uint32_t n0 = nt * BN;
    const uint64_t sp0 = uint64_t(ks) * a.sps;
    const uint32_t nsp = uint32_t(umin64(a.nspans, sp0 + a.sps) - sp0);
    const uint64_t k0 = sp0 * kGmSpan, k1 = umin64(a.cols, k0 + uint64_t(nsp) * kGmSpan);
    const uint32_t nkb = uint32_t((k1 - k0 + kGmKB - 1) / kGmKB);

    init_luts(tid);
    if (tid == 0) {
        for (int s = 0; s < C::kXS; ++s) {
            mbar_init(xfull0 + 8 * s, 1);                     // X expect_tx
            mbar_init(xempty0 + 8 * s, 1);                    // tcgen05.commit
        }
        for (int s = 0; s < kGmAS; ++s) {
            mbar_init(afull0 + 8 * s, kGmExpandWarps / 2);    // the 8 warps of a k-block parity
            mbar_init(aempty0 + 8 * s, 1);                    // tcgen05.commit
        }
        for (int s = 0; s < kGmBmp; ++s) {
            mbar_init(bfull0 + 8 * s, 32);                    // bitmap producer lanes
            mbar_init(bempty0 + 8 * s, kGmExpandWarps);
        }
        mbar_init(tfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
    }
    pdl_wait();  // idx (count + flatten) and the latched status come from the previous kernels
    if (cta_error_latched(a.hdr)) return;
    pdl_launch_dependents();
    if (warp == 2) {  // TMEM accumulator: BN fp32 columns x 128 lanes
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sb + C::kTmemSlot),
                     "r"(C::kTmemCols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // row value cursors at the split's range ends (every warp takes rows)
    for (int r = warp; r < kGmRows; r += kGmThreads / 32) {
        const uint64_t gr = m0 + r;
        unsigned long long s0 = 0, s1 = 0;
        if (gr < a.rows) {
            const uint64_t p0 = gr * a.cols + k0, p1 = gr * a.cols + k1;
            s0 = warp_rank(a, p0, lane);
            s1 = p1 >= a.rows * a.cols ? a.nnz : warp_rank(a, p1, lane);
        }
        if (lane == 0) {
            rstart[r] = s0;
            rend[r] = s1;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + C::kTmemSlot);

    if (warp == 0) {
        // ===== bitmap producer: 16 bytes per row per 128-column span, kGmBmp spans ahead =====
        for (uint32_t sn = 0; sn < nsp; ++sn) {
            const uint32_t bs = sn % kGmBmp;
            mbar_wait(bempty0 + 8 * bs, ((sn / kGmBmp) & 1) ^ 1);
            const uint32_t bslot = sb + C::kBmpOff + bs * kGmBmpBytes;
            const uint64_t kc = k0 + uint64_t(sn) * kGmSpan;
            if (a.bmp_async) {  // cols % 128 == 0, 16-byte aligned bitmap: 16 aligned bytes per row
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int r = lane + 32 * i;
                    const bool live = m0 + r < a.rows;
                    const uint8_t* src = a.bitmap + (live ? ((m0 + r) * a.cols + kc) / 8 : 0);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(bslot + r * 16), "l"(src),
                                 "r"(live ? 16 : 0) : "memory");
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bfull0 + 8 * bs) : "memory");
            } else {  // any cols: 128 bits from bit (gr*cols + kc), funnel-shifted, masked to the range
                const uint32_t valid = uint32_t(umin64(kGmSpan, k1 - kc));
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int r = lane + 32 * i;
                    uint4 q = make_uint4(0, 0, 0, 0);
                    if (m0 + r < a.rows) {
                        const uint64_t b = (m0 + r) * a.cols + kc, w = b >> 5;
                        const uint32_t sh = uint32_t(b & 31);
                        uint32_t wd[5];
#pragma unroll
                        for (int t = 0; t < 5; ++t) wd[t] = load_word32(a.bitmap, w + t, a.nbytes);
                        uint32_t o[4];
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            o[t] = __funnelshift_r(wd[t], wd[t + 1], sh);
                            const int lo = 32 * t;
                            if (int(valid) <= lo) o[t] = 0;
                            else if (int(valid) < lo + 32) o[t] &= (1u << (valid - lo)) - 1u;
                        }
                        q = make_uint4(o[0], o[1], o[2], o[3]);
                    }
                    sts128(bslot + r * 16, q);
                }
                mbar_arrive(bfull0 + 8 * bs);
            }
        }
    } else if (warp == 1) {
        // ===== X producer =====
        if (lane == 0)
            for (uint32_t kb = 0; kb < nkb; ++kb) {
                const uint32_t st = kb % C::kXS;
                mbar_wait(xempty0 + 8 * st, ((kb / C::kXS) & 1) ^ 1);
                mbar_arrive_expect_tx(xfull0 + 8 * st, BN * 128);
                tma_load_2d(sb + C::kB + st * (BN * 128), &xmap, int(k0 + uint64_t(kb) * kGmKB), int(n0),
                            xfull0 + 8 * st);
            }
    } else if (warp == 2) {
        // ===== MMA issuer: A (the expanded W rows) from TMEM, X from shared memory =====
        // kind::f16: D f32 (bit 4), A = B = f16, both K-major, N >> 3 at bit 17, M >> 4 at bit 24
        constexpr uint32_t idesc = (1u << 4) | (uint32_t(BN >> 3) << 17) | (uint32_t(kGmRows >> 4) << 24);
        for (uint32_t kb = 0; kb < nkb; ++kb) {
            const uint32_t sx = kb % C::kXS, sa = kb % kGmAS;
            mbar_wait(xfull0 + 8 * sx, (kb / C::kXS) & 1);
            mbar_wait(afull0 + 8 * sa, (kb / kGmAS) & 1);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t at = tmem + BN + 32 * sa;  // A stage: lane = W row, 2 f16 per column
                const uint64_t bd = umma_desc_sw128(sb + C::kB + sx * (BN * 128));
#pragma unroll
                for (int k = 0; k < kGmKB / 16; ++k)  // K = 16: 8 A columns, +32 bytes of X per step
                    if (!(ENDOR_GEMM_SKIP & 1)) umma_f16_ts(tmem, at + 8 * k, bd + 2 * k, idesc, (kb | k) != 0);
                umma_commit(xempty0 + 8 * sx);
                umma_commit(aempty0 + 8 * sa);
                if (kb + 1 == nkb) umma_commit(tfull);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ===== expand: thread (row r, k-block parity h, half c2) fills 32
        // columns of row r of every k-block 2s + h.  It copies its own values
        // window of span s + kLook (16-byte cp.async into a private slot) while
        // expanding span s, so no other thread touches its raw bytes. =====
        const int ew = warp - 4;          // expand warp 0..15
        const int q = warp & 3;           // TMEM lane quadrant this warp may access
        const int h = (ew >> 2) & 1;      // k-block parity: 0 = even, 1 = odd k-blocks
        const int c2 = ew >> 3;           // which 32 columns of the k-block
        const int wsel = 2 * h + c2;      // bitmap word of the span (32 columns each)
        const int r = 32 * q + lane;      // W row within the tile
        const int et = tid - 4 * 32;      // expand thread 0..511
        const uint64_t vlo = reinterpret_cast<uint64_t>(a.values), vhi = vlo + a.nnz * 2;
        const uint64_t safe_lo = (vlo + 15) & ~uint64_t(15), safe_hi = vhi & ~uint64_t(15);
        const uint32_t win0 = sb + C::kRawOff + et * kGmWin;  // + slot * kGmRawBytes
        unsigned long long icur = rstart[r], gcur = icur;      // issue / gather cursors (value index)
        const unsigned long long iend = rend[r];
        bool bad = icur > iend || iend > a.nnz;
        auto word = [](const uint4& b, int i) { return i == 0 ? b.x : (i == 1 ? b.y : (i == 2 ? b.z : b.w)); };
        auto before = [&](const uint4& b) {  // set bits of the span ahead of this thread's 32 columns
            uint32_t n = 0;
#pragma unroll
            for (int i = 0; i < 3; ++i) n += i < wsel ? __popc(word(b, i)) : 0u;
            return n;
        };
        // copy this thread's window of span sn into slot sn % kRaw
        auto issue = [&](uint32_t sn) {
            const uint32_t bs = sn % kGmBmp;
            mbar_wait(bfull0 + 8 * bs, (sn / kGmBmp) & 1);
            const uint4 bits = lds128(sb + C::kBmpOff + bs * kGmBmpBytes + r * 16);
            unsigned long long c0 = icur + before(bits), c1 = c0 + __popc(word(bits, wsel));
            icur += __popc(bits.x) + __popc(bits.y) + __popc(bits.z) + __popc(bits.w);
            if (c1 > a.nnz) {
                bad = true;
                c1 = a.nnz;
                c0 = c0 < c1 ? c0 : c1;
            }
            if (c1 <= c0) return;
            const uint64_t a0 = vlo + 2 * c0, a1 = vlo + 2 * c1;
            const uint64_t A0 = a0 & ~uint64_t(15), A1 = (a1 + 15) & ~uint64_t(15);
            const uint32_t dst = win0 + (sn % C::kRaw) * kGmRawBytes;
            if (ENDOR_GEMM_SKIP & 4) return;
            if (A0 >= safe_lo && A1 <= safe_hi) {
                for (uint64_t p = A0; p < A1; p += 16)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + uint32_t(p - A0)), "l"(p)
                                 : "memory");
            } else {  // a window touching a ragged end of the values buffer: bytewise
                for (uint64_t p = a0; p < a1; ++p) sts8(dst + uint32_t(p - A0), *reinterpret_cast<const uint8_t*>(p));
            }
        };
        for (uint32_t sn = 0; sn < uint32_t(C::kLook); ++sn) {
            if (sn < nsp) issue(sn);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        for (uint32_t s = 0; s < nsp; ++s) {
            if (s + C::kLook < nsp) issue(s + C::kLook);
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group %0;" ::"n"(C::kLook) : "memory");  // span s's copies landed
            const uint32_t bs = s % kGmBmp;
            const uint4 bits = lds128(sb + C::kBmpOff + bs * kGmBmpBytes + r * 16);
            __syncwarp();
            if (lane == 0) mbar_arrive(bempty0 + 8 * bs);  // this warp is done with span s's bitmap
            const uint32_t kb = 2 * s + h;
            const uint32_t m32 = word(bits, wsel);
            const unsigned long long c0 = gcur + before(bits);
            gcur += __popc(bits.x) + __popc(bits.y) + __popc(bits.z) + __popc(bits.w);
            if (kb >= nkb) continue;  // ragged last span: no odd k-block
            const uint32_t sa = kb % kGmAS;
            uint32_t ca = win0 + (s % C::kRaw) * kGmRawBytes + uint32_t((vlo + 2 * c0) & 15);
            // all four gathers first (their LDS issue back to back), then one TMEM store
            uint4 v[4];
            if (!(ENDOR_GEMM_SKIP & 2))
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t m = (m32 >> (8 * c)) & 0xFFu;
                v[c] = gather_chunk<2>(m, ca);
                ca += 2 * __popc(m);
            }
            if (ENDOR_GEMM_SKIP & 2)
                for (int c = 0; c < 4; ++c) v[c] = make_uint4(m32, ca, c, 0);
            mbar_wait(aempty0 + 8 * sa, ((kb / kGmAS) & 1) ^ 1);
            tc_fence_after();
            tmem_st16(tmem + (uint32_t(32 * q) << 16) + BN + 32 * sa + 16 * c2, v);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(afull0 + 8 * sa);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        if (m0 + r < a.rows && icur != iend) bad = true;
        if (bad) latch_status(a.hdr, ENDOR_ERR_CORRUPTION);
        // ---- epilogue: TMEM -> registers -> Y (or the split's fp32 partial) ----
        mbar_wait(tfull, 0);
        tc_fence_after();
        const uint64_t gr = m0 + r;
        constexpr int kQuarter = BN / 4;  // columns per expand warp of this lane quadrant
        const int col0 = (ew >> 2) * kQuarter;
#pragma unroll 1
        for (int c0 = 0; c0 < kQuarter; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(tmem + (uint32_t(32 * q) << 16) + uint32_t(col0 + c0), v);
            if (gr < a.rows) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const uint64_t n = uint64_t(n0) + col0 + c0 + i;
                    if (n < a.tokens) {
                        const float f = __uint_as_float(v[i]);
                        if (a.ksplit > 1) {
                            a.part[(uint64_t(ks) * a.tokens + n) * a.rows + gr] = f;
                        } else {
                            if (a.y32) a.y32[n * a.rows + gr] = f;
                            if (a.y16) a.y16[n * a.rows + gr] = __float2half_rn(f);
                        }
                    }
                }
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kTmemCols) : "memory");
    }
}

// ---------------------------------------------------------------------------------
// Dense GEMM consumer (the two-pass path for large token counts, and
// endor_cuda_gemm): Y = X W^T with W already decompressed in HBM.  A canonical
// tcgen05 pipeline: one TMA warp loads each k-block's 128 x 64 W tile and BN x 64
// X tile (128-byte swizzle) into a kDS-deep ring, one elected lane issues 4 SS
// MMAs per k-block into a TMEM accumulator, four epilogue warps drain it.
// ---------------------------------------------------------------------------------
constexpr int kGdThreads = 256;
template <int BN>
struct GdCfg {
    static constexpr int kStage = 16384 + BN * 128;
    static constexpr int kDS = (200 * 1024) / kStage;             // 4 (BN 256), 6 (128), 8 (64)
    static constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
    static constexpr uint32_t kBar = kDS * kStage;
    static constexpr uint32_t kTmemSlot = kBar + 8 * (2 * kDS + 1);
    static constexpr uint32_t kSmem = kTmemSlot + 16 + 1024;
};

template <int BN>
__global__ void __launch_bounds__(kGdThreads, 1)
    gemm_dense_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap xmap,
                      const __grid_constant__ GemmArgs a) {
    using C = GdCfg<BN>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t sraw = smem_u32(smem_raw);
    const uint32_t sb = (sraw + 1023u) & ~1023u;
    uint8_t* const smem = smem_raw + (sb - sraw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t full0 = sb + C::kBar, empty0 = full0 + 8 * C::kDS, tfull = empty0 + 8 * C::kDS;
    uint32_t u = blockIdx.x;
    const uint32_t nt = u % a.n_tiles;
    u /= a.n_tiles;
    const uint32_t ks = u % a.ksplit, mt = u / a.ksplit;
    const uint64_t m0 = uint64_t(mt) * kGmRows;
    const uint32_t n0 = nt * BN;
    const uint64_t sp0 = uint64_t(ks) * a.sps;
    const uint32_t nsp = uint32_t(umin64(a.nspans, sp0 + a.sps) - sp0);
    const uint64_t k0 = sp0 * kGmSpan, k1 = umin64(a.cols, k0 + uint64_t(nsp) * kGmSpan);
    const uint32_t nkb = uint32_t((k1 - k0 + kGmKB - 1) / kGmKB);
    if (tid == 0) {
        for (int s = 0; s < C::kDS; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        mbar_init(tfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
    }
    pdl_wait();  // W comes from the decompress launch before this one
    if (cta_error_latched(a.hdr)) return;
    pdl_launch_dependents();
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sb + C::kTmemSlot),
                     "r"(C::kTmemCols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + C::kTmemSlot);
    if (warp == 0) {
        if (lane == 0)
            for (uint32_t kb = 0; kb < nkb; ++kb) {
                const uint32_t st = kb % C::kDS;
                mbar_wait(empty0 + 8 * st, ((kb / C::kDS) & 1) ^ 1);
                mbar_arrive_expect_tx(full0 + 8 * st, C::kStage);
                const int kc = int(k0 + uint64_t(kb) * kGmKB);
                tma_load_2d(sb + st * C::kStage, &wmap, kc, int(m0), full0 + 8 * st);
                tma_load_2d(sb + st * C::kStage + 16384, &xmap, kc, int(n0), full0 + 8 * st);
            }
    } else if (warp == 1) {
        constexpr uint32_t idesc = (1u << 4) | (uint32_t(BN >> 3) << 17) | (uint32_t(kGmRows >> 4) << 24);
        for (uint32_t kb = 0; kb < nkb; ++kb) {
            const uint32_t st = kb % C::kDS;
            mbar_wait(full0 + 8 * st, (kb / C::kDS) & 1);
            tc_fence_after();
            if (lane == 0) {
                const uint64_t ad = umma_desc_sw128(sb + st * C::kStage);
                const uint64_t bd = umma_desc_sw128(sb + st * C::kStage + 16384);
#pragma unroll
                for (int k = 0; k < kGmKB / 16; ++k) umma_f16(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
                umma_commit(empty0 + 8 * st);
                if (kb + 1 == nkb) umma_commit(tfull);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        const int q = warp & 3, r = 32 * q + lane;
        const uint64_t gr = m0 + r;
        mbar_wait(tfull, 0);
        tc_fence_after();
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(tmem + (uint32_t(32 * q) << 16) + uint32_t(c0), v);
            if (gr < a.rows) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const uint64_t n = uint64_t(n0) + c0 + i;
                    if (n < a.tokens) {
                        const float f = __uint_as_float(v[i]);
                        if (a.ksplit > 1) {
                            a.part[(uint64_t(ks) * a.tokens + n) * a.rows + gr] = f;
                        } else {
                            if (a.y32) a.y32[n * a.rows + gr] = f;
                            if (a.y16) a.y16[n * a.rows + gr] = __float2half_rn(f);
                        }
                    }
                }
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kTmemCols) : "memory");
    }
}

// split-K: Y = sum over splits of the fp32 partials, in split order (deterministic)
__global__ void __launch_bounds__(256) gemm_reduce_kernel(const float* __restrict__ part, uint64_t count,
                                                          uint32_t ksplit, float* y32, __half* y16,
                                                          const WsHeader* hdr) {
    pdl_wait();
    if (read_status(hdr)) return;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += uint64_t(gridDim.x) * blockDim.x) {
        float s = 0.f;
        for (uint32_t k = 0; k < ksplit; ++k) s += __ldcs(part + uint64_t(k) * count + i);
        if (y32) y32[i] = s;
        if (y16) y16[i] = __float2half_rn(s);
    }
}

// ---- host side ------------------------------------------------------------------
GemmPlan gemm_plan(uint64_t rows, uint64_t cols, uint64_t tokens, int sms) {
    GemmPlan p{};
    p.bn = tokens <= 64 ? 64 : (tokens <= 128 ? 128 : 256);
    p.m_tiles = uint32_t(ceil_div(rows, kGmRows));
    p.n_tiles = uint32_t(ceil_div(tokens, p.bn));
    p.nspans = ceil_div(cols, kGmSpan);
    // split K until the grid fills the SMs (one CTA per SM), in whole waves
    const uint64_t base = uint64_t(p.m_tiles) * p.n_tiles;
    uint32_t best = 1;
    double best_eff = 0;
    for (uint32_t k = 1; k <= 16 && k <= p.nspans; ++k) {
        const uint64_t sps = ceil_div(p.nspans, k), kk = ceil_div(p.nspans, sps);
        const uint64_t units = base * kk, waves = ceil_div(units, uint64_t(sms));
        const double eff = double(units) / double(waves * sms);
        if (eff > best_eff * 1.05) {  // a further split must buy > 5 %
            best_eff = eff;
            best = uint32_t(kk);
        }
        if (base * k >= uint64_t(sms)) break;
    }
    p.sps = uint32_t(ceil_div(p.nspans, best));
    p.ksplit = uint32_t(ceil_div(p.nspans, p.sps));
    p.part_bytes = p.ksplit > 1 ? p.ksplit * tokens * rows * 4 : 0;
    // Large token counts: the fused kernel re-expands each W tile once per
    // 256-token n-tile, so past ~384 tokens decompressing W once into HBM (at
    // the copy roofline) and running the dense tcgen05 GEMM wins (fc1: fused
    // 0.52 vs 0.45 ms at 512 tokens, 1.91 vs 1.12 ms at 2048; profiles/r02).
    static const uint64_t two_pass_tokens = [] {
        const char* e = getenv("ENDOR_GEMM_TWO_PASS_TOKENS");
        return e ? uint64_t(strtoull(e, nullptr, 10)) : uint64_t(384);
    }();
    p.two_pass = tokens > two_pass_tokens && cols % 8 == 0;
    return p;
}

namespace {
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled encode_fn() {
    static EncodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiled>(p);
    });
    return fn;
}
}  // namespace

template <int BN>
static cudaError_t launch_bn(const GemmPlan& p, const CUtensorMap& xm, const GemmArgs& a, cudaStream_t s) {
    int bps = 1, sms = 148;
    cudaError_t e = kernel_slots(reinterpret_cast<const void*>(gemm_fused_kernel<BN>), kGmThreads, GmCfg<BN>::kSmem,
                                 &bps, &sms);
    if (e != cudaSuccess) return e;
    const uint64_t units = uint64_t(p.m_tiles) * p.n_tiles * p.ksplit;
    return launch_pdl(gemm_fused_kernel<BN>, dim3(unsigned(units)), dim3(kGmThreads), GmCfg<BN>::kSmem, s, xm, a);
}

template <int BN>
static cudaError_t launch_dense(const GemmPlan& p, const CUtensorMap& wm, const CUtensorMap& xm, const GemmArgs& a,
                                cudaStream_t s) {
    int bps = 1, sms = 148;
    cudaError_t e = kernel_slots(reinterpret_cast<const void*>(gemm_dense_kernel<BN>), kGdThreads, GdCfg<BN>::kSmem,
                                 &bps, &sms);
    if (e != cudaSuccess) return e;
    const uint64_t units = uint64_t(p.m_tiles) * p.n_tiles * p.ksplit;
    return launch_pdl(gemm_dense_kernel<BN>, dim3(unsigned(units)), dim3(kGdThreads), GdCfg<BN>::kSmem, s, wm, xm, a);
}

cudaError_t launch_gemm_fused(const GemmPlan& p, const GemmLaunch& g, cudaStream_t s) {
    EncodeTiled enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap xm{};
    {
        const cuuint64_t dims[2] = {g.cols, g.tokens};
        const cuuint64_t strides[1] = {g.x_ld * 2};
        const cuuint32_t box[2] = {uint32_t(kGmKB), uint32_t(p.bn)}, es[2] = {1, 1};
        if (enc(&xm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(g.x), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    const bool bmp_async = g.cols % kGmSpan == 0 && (reinterpret_cast<uintptr_t>(g.bitmap) & 15) == 0;
    GemmArgs a{};
    a.bitmap = g.bitmap;
    a.nbytes = (g.rows * g.cols + 7) / 8;
    a.values = g.values;
    a.nnz = g.nnz;
    a.idx = g.idx;
    a.rows = g.rows;
    a.cols = g.cols;
    a.tokens = g.tokens;
    a.m_tiles = p.m_tiles;
    a.n_tiles = p.n_tiles;
    a.ksplit = p.ksplit;
    a.sps = p.sps;
    a.nspans = p.nspans;
    a.part = g.part;
    a.y32 = g.y32;
    a.y16 = reinterpret_cast<__half*>(g.y16);
    a.hdr = g.hdr;
    a.bmp_async = bmp_async ? 1 : 0;
    cudaError_t e;
    if (g.w_dense) {
        CUtensorMap wm{};
        const cuuint64_t dims[2] = {g.cols, g.rows};
        const cuuint64_t strides[1] = {g.cols * 2};
        const cuuint32_t box[2] = {uint32_t(kGmKB), uint32_t(kGmRows)}, es[2] = {1, 1};
        if (enc(&wm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(g.w_dense), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
        e = p.bn == 64    ? launch_dense<64>(p, wm, xm, a, s)
            : p.bn == 128 ? launch_dense<128>(p, wm, xm, a, s)
                          : launch_dense<256>(p, wm, xm, a, s);
    } else {
        e = p.bn == 64    ? launch_bn<64>(p, xm, a, s)
            : p.bn == 128 ? launch_bn<128>(p, xm, a, s)
                          : launch_bn<256>(p, xm, a, s);
    }
    if (e != cudaSuccess || p.ksplit <= 1) return e;
    const uint64_t count = g.tokens * g.rows;
    const unsigned blocks = unsigned(umin64(ceil_div(count, 256), 148 * 8));
    return launch_pdl(gemm_reduce_kernel, dim3(blocks), dim3(256), 0, s, static_cast<const float*>(g.part), count,
                      p.ksplit, g.y32, reinterpret_cast<__half*>(g.y16), static_cast<const WsHeader*>(g.hdr));
}

}  // namespace endor_b200
