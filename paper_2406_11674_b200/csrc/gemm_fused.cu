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
//   warp 0      raw producer: per 128-column span, the span's bitmap (16 bytes
//               per row; 2-D TMA when cols % 128 == 0) and every row's packed
//               values window (one 1-D bulk copy per row, 16-byte aligned
//               superset) into a raw ring; row value cursors advance by popc
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

#include <mutex>

#include "common.cuh"
#include "gather.cuh"
#include "kernels.h"

namespace endor_b200 {

constexpr int kGmRows = 128;                        // UMMA M
constexpr int kGmKB = 64;                           // k-block: 64 f16 = one 128-byte swizzle row
constexpr int kGmSpan = 128;                        // raw stage: 2 k-blocks, 16 bitmap bytes per row
constexpr int kGmSlotRow = 272;                     // <= 128 values + 16-byte alignment slack
constexpr int kGmRawHdr = kGmRows * 4;              // per-row byte offset of the first value
constexpr int kGmRawBytes = kGmRawHdr + kGmRows * kGmSlotRow;  // 35328
constexpr int kGmBmpBytes = kGmRows * 16;           // 2048
constexpr int kGmExpandWarps = 8;
constexpr int kGmThreads = (4 + kGmExpandWarps) * 32;  // 384

template <int BN>
struct GmCfg {
    static constexpr int kAB = BN == 256 ? 3 : 4;                 // A/B stages
    static constexpr int kRaw = BN == 64 ? 3 : 2;                 // raw (values) stages
    static constexpr int kBmp = BN == 256 ? 4 : 8;                // bitmap stages (lookahead kBmp - kRaw spans)
    static constexpr uint32_t kA = 0;                             // A tiles, 16 KiB each (1024-aligned)
    static constexpr uint32_t kB = kA + kAB * 16384;              // X tiles, BN x 128 bytes
    static constexpr uint32_t kRawOff = kB + kAB * BN * 128;
    static constexpr uint32_t kBmpOff = kRawOff + kRaw * kGmRawBytes;
    static constexpr uint32_t kBar = kBmpOff + kBmp * kGmBmpBytes;
    // full[kAB] empty[kAB] raw_full[kRaw] raw_empty[kRaw] bmp_full[kBmp] tmem_full, tmem addr
    static constexpr uint32_t kTmemSlot = kBar + 8 * (2 * kAB + 2 * kRaw + kBmp + 1);
    static constexpr uint32_t kRank = (kTmemSlot + 4 + 15) & ~15u;  // u64 start[128], end[128]
    static constexpr uint32_t kEnd = kRank + 2 * 8 * kGmRows + 16;  // + gather over-read pad
    static constexpr uint32_t kSmem = kEnd + 1024;                  // + alignment of the dynamic base
};
static_assert(GmCfg<256>::kSmem <= 232448 && GmCfg<128>::kSmem <= 232448 && GmCfg<64>::kSmem <= 232448,
              "GEMM shared-memory plan exceeds 227 KiB");

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
    int bmp_tma;                             // bitmap via the 2-D tensor map
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
    gemm_fused_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap bmap,
                      const __grid_constant__ GemmArgs a) {
    using C = GmCfg<BN>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t sraw = smem_u32(smem_raw);
    const uint32_t sb = (sraw + 1023u) & ~1023u;  // swizzle-128B operands need 1024-byte alignment
    uint8_t* const smem = smem_raw + (sb - sraw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    const uint32_t full0 = sb + C::kBar, empty0 = full0 + 8 * C::kAB;
    const uint32_t rfull0 = empty0 + 8 * C::kAB, rempty0 = rfull0 + 8 * C::kRaw;
    const uint32_t bfull0 = rempty0 + 8 * C::kRaw, tfull = bfull0 + 8 * C::kBmp;
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
        for (int s = 0; s < C::kAB; ++s) {
            mbar_init(full0 + 8 * s, 1 + kGmExpandWarps);  // X expect_tx + the expand warps
            mbar_init(empty0 + 8 * s, 1);                 // tcgen05.commit
        }
        for (int s = 0; s < C::kRaw; ++s) {
            mbar_init(rfull0 + 8 * s, 32);                // every producer lane (expect_tx)
            mbar_init(rempty0 + 8 * s, kGmExpandWarps);
        }
        for (int s = 0; s < C::kBmp; ++s) mbar_init(bfull0 + 8 * s, 1);
        mbar_init(tfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
        if (a.bmp_tma) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap)) : "memory");
    }
    pdl_wait();  // idx (count + flatten) and the latched status come from the previous kernels
    if (cta_error_latched(a.hdr)) return;
    pdl_launch_dependents();
    if (warp == 2) {  // TMEM accumulator: BN fp32 columns x 128 lanes
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sb + C::kTmemSlot),
                     "r"(uint32_t(BN)) : "memory");
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
        // ===== raw producer: bitmap spans + per-row value windows =====
        constexpr int kLookBmp = C::kBmp - C::kRaw;  // bitmap spans in flight beyond the raw ring
        const uint64_t vlo = reinterpret_cast<uint64_t>(a.values), vhi = vlo + a.nnz * 2;
        const uint64_t safe_lo = (vlo + 15) & ~uint64_t(15), safe_hi = vhi & ~uint64_t(15);
        unsigned long long cur[4];
        bool bad = false;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            cur[i] = rstart[lane + 32 * i];
            bad |= cur[i] > rend[lane + 32 * i] || rend[lane + 32 * i] > a.nnz;
        }
        if (a.bmp_tma && lane == 0)
            for (uint32_t s = 0; s < nsp && s < uint32_t(kLookBmp); ++s) {
                mbar_arrive_expect_tx(bfull0 + 8 * s, kGmBmpBytes);
                tma_load_2d(sb + C::kBmpOff + s * kGmBmpBytes, &bmap, int((sp0 + s) * 16), int(m0), bfull0 + 8 * s);
            }
        for (uint32_t s = 0; s < nsp; ++s) {
            const uint32_t rs = s % C::kRaw, bs = s % C::kBmp;
            mbar_wait(rempty0 + 8 * rs, ((s / C::kRaw) & 1) ^ 1);
            const uint32_t bslot = sb + C::kBmpOff + bs * kGmBmpBytes;
            if (a.bmp_tma) {
                const uint32_t sn = s + kLookBmp;
                if (lane == 0 && sn < nsp) {
                    const uint32_t bn = sn % C::kBmp;
                    mbar_arrive_expect_tx(bfull0 + 8 * bn, kGmBmpBytes);
                    tma_load_2d(sb + C::kBmpOff + bn * kGmBmpBytes, &bmap, int((sp0 + sn) * 16), int(m0),
                                bfull0 + 8 * bn);
                }
                mbar_wait(bfull0 + 8 * bs, (s / C::kBmp) & 1);
            } else {
                // generic: any cols -- 128 bits from bit (gr*cols + k), funnel-shifted, masked to the range
                const uint64_t kc = k0 + uint64_t(s) * kGmSpan;
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
            }
            const uint32_t raw = sb + C::kRawOff + rs * kGmRawBytes;
            uint32_t bytes = 0;
            uint64_t src[4];
            uint32_t len[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int r = lane + 32 * i;
                const uint4 q = lds128(bslot + r * 16);
                const uint32_t pc = __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
                unsigned long long c0 = cur[i], c1 = c0 + pc;
                if (c1 > a.nnz) {
                    bad = true;
                    c1 = a.nnz;
                    c0 = c0 < c1 ? c0 : c1;
                }
                cur[i] = c1;
                const uint64_t a0 = vlo + 2 * c0, a1 = vlo + 2 * c1;
                const uint64_t A0 = a0 & ~uint64_t(15), A1 = (a1 + 15) & ~uint64_t(15);
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(raw + 4 * r), "r"(uint32_t(a0 - A0)) : "memory");
                src[i] = A0;
                len[i] = 0;
                if (c1 > c0) {
                    if (A0 >= safe_lo && A1 <= safe_hi) {
                        len[i] = uint32_t(A1 - A0);
                        bytes += len[i];
                    } else {  // a window touching a ragged end of the values buffer: bytewise
                        const uint32_t dst = raw + kGmRawHdr + r * kGmSlotRow;
                        for (uint64_t p = a0; p < a1; ++p)
                            sts8(dst + uint32_t(p - A0), *reinterpret_cast<const uint8_t*>(p));
                        fence_proxy_async_smem();  // a later bulk copy overwrites these bytes
                    }
                }
            }
            mbar_arrive_expect_tx(rfull0 + 8 * rs, bytes);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (len[i])
                    bulk_g2s(raw + kGmRawHdr + (lane + 32 * i) * kGmSlotRow, reinterpret_cast<const void*>(src[i]),
                             len[i], rfull0 + 8 * rs);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (m0 + lane + 32 * i < a.rows) bad |= cur[i] != rend[lane + 32 * i];
        if (bad) latch_status(a.hdr, ENDOR_ERR_CORRUPTION);
    } else if (warp == 1) {
        // ===== X producer =====
        if (lane == 0)
            for (uint32_t kb = 0; kb < nkb; ++kb) {
                const uint32_t st = kb % C::kAB;
                mbar_wait(empty0 + 8 * st, ((kb / C::kAB) & 1) ^ 1);
                mbar_arrive_expect_tx(full0 + 8 * st, BN * 128);
                tma_load_2d(sb + C::kB + st * (BN * 128), &xmap, int(k0 + uint64_t(kb) * kGmKB), int(n0),
                            full0 + 8 * st);
            }
    } else if (warp == 2) {
        // ===== MMA issuer =====
        // kind::f16: D f32 (bit 4), A = B = f16, both K-major, N >> 3 at bit 17, M >> 4 at bit 24
        constexpr uint32_t idesc = (1u << 4) | (uint32_t(BN >> 3) << 17) | (uint32_t(kGmRows >> 4) << 24);
        for (uint32_t kb = 0; kb < nkb; ++kb) {
            const uint32_t st = kb % C::kAB;
            mbar_wait(full0 + 8 * st, (kb / C::kAB) & 1);
            tc_fence_after();
            if (lane == 0) {
                const uint64_t ad = umma_desc_sw128(sb + C::kA + st * 16384);
                const uint64_t bd = umma_desc_sw128(sb + C::kB + st * (BN * 128));
#pragma unroll
                for (int k = 0; k < kGmKB / 16; ++k)  // +32 bytes per K = 16 step inside the swizzle atom
                    umma_f16(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
                umma_commit(empty0 + 8 * st);
                if (kb + 1 == nkb) umma_commit(tfull);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ===== expand into the A stage, then the epilogue =====
        const int q = warp & 3;           // TMEM lane quadrant this warp may access
        const int h = (warp - 4) >> 2;    // which 4 of the k-block's 8 chunks
        const int r = 32 * q + lane;      // W row within the tile
        const uint32_t sw = uint32_t(r & 7);
        for (uint32_t s = 0; s < nsp; ++s) {
            const uint32_t rs = s % C::kRaw;
            mbar_wait(rfull0 + 8 * rs, (s / C::kRaw) & 1);
            const uint32_t raw = sb + C::kRawOff + rs * kGmRawBytes;
            const uint4 bits = lds128(sb + C::kBmpOff + (s % C::kBmp) * kGmBmpBytes + r * 16);
            uint32_t va = raw + kGmRawHdr + r * kGmSlotRow + lds32(raw + 4 * r);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t kb = 2 * s + j;
                if (kb >= nkb) break;
                const uint32_t lo = j ? bits.z : bits.x, hi = j ? bits.w : bits.y;
                const uint32_t st = kb % C::kAB;
                const uint32_t m32 = h ? hi : lo;
                uint32_t ca = va + (h ? 2 * __popc(lo) : 0);
                va += 2 * (__popc(lo) + __popc(hi));
                mbar_wait(empty0 + 8 * st, ((kb / C::kAB) & 1) ^ 1);
                const uint32_t arow = sb + C::kA + st * 16384 + r * 128;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const uint32_t m = (m32 >> (8 * c)) & 0xFFu;
                    const uint4 v = gather_chunk<2>(m, ca);
                    ca += 2 * __popc(m);
                    sts128(arow + ((uint32_t(4 * h + c) ^ sw) << 4), v);
                }
                fence_proxy_async_smem();  // generic-proxy A writes -> the tensor core's async-proxy reads
                __syncwarp();
                if (lane == 0) mbar_arrive(full0 + 8 * st);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(rempty0 + 8 * rs);
        }
        // ---- epilogue: TMEM -> registers -> Y (or the split's fp32 partial) ----
        mbar_wait(tfull, 0);
        tc_fence_after();
        const uint64_t gr = m0 + r;
        constexpr int kHalf = BN / 2;
#pragma unroll 1
        for (int c0 = 0; c0 < kHalf; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(tmem + (uint32_t(32 * q) << 16) + uint32_t(h * kHalf + c0), v);
            if (gr < a.rows) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const uint64_t n = uint64_t(n0) + h * kHalf + c0 + i;
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
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(uint32_t(BN)) : "memory");
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
static cudaError_t launch_bn(const GemmPlan& p, const GemmLaunch& g, const CUtensorMap& xm, const CUtensorMap& bm,
                             const GemmArgs& a, cudaStream_t s) {
    int bps = 1, sms = 148;
    cudaError_t e = kernel_slots(reinterpret_cast<const void*>(gemm_fused_kernel<BN>), kGmThreads, GmCfg<BN>::kSmem,
                                 &bps, &sms);
    if (e != cudaSuccess) return e;
    const uint64_t units = uint64_t(p.m_tiles) * p.n_tiles * p.ksplit;
    (void)g;
    return launch_pdl(gemm_fused_kernel<BN>, dim3(unsigned(units)), dim3(kGmThreads), GmCfg<BN>::kSmem, s, xm, bm, a);
}

cudaError_t launch_gemm_fused(const GemmPlan& p, const GemmLaunch& g, cudaStream_t s) {
    EncodeTiled enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap xm{}, bm{};
    {
        const cuuint64_t dims[2] = {g.cols, g.tokens};
        const cuuint64_t strides[1] = {g.x_ld * 2};
        const cuuint32_t box[2] = {uint32_t(kGmKB), uint32_t(p.bn)}, es[2] = {1, 1};
        if (enc(&xm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(g.x), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    const bool bmp_tma = g.cols % kGmSpan == 0 && (reinterpret_cast<uintptr_t>(g.bitmap) & 15) == 0;
    if (bmp_tma) {
        const cuuint64_t dims[2] = {g.cols / 8, g.rows};
        const cuuint64_t strides[1] = {g.cols / 8};
        const cuuint32_t box[2] = {16, uint32_t(kGmRows)}, es[2] = {1, 1};
        if (enc(&bm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(g.bitmap), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
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
    a.bmp_tma = bmp_tma ? 1 : 0;
    cudaError_t e = p.bn == 64    ? launch_bn<64>(p, g, xm, bm, a, s)
                    : p.bn == 128 ? launch_bn<128>(p, g, xm, bm, a, s)
                                  : launch_bn<256>(p, g, xm, bm, a, s);
    if (e != cudaSuccess || p.ksplit <= 1) return e;
    const uint64_t count = g.tokens * g.rows;
    const unsigned blocks = unsigned(umin64(ceil_div(count, 256), 148 * 8));
    return launch_pdl(gemm_reduce_kernel, dim3(blocks), dim3(256), 0, s, static_cast<const float*>(g.part), count,
                      p.ksplit, g.y32, reinterpret_cast<__half*>(g.y16), static_cast<const WsHeader*>(g.hdr));
}

}  // namespace endor_b200
