// gemv_fused.cu -- fused decompress -> GEMV: y = W x straight from the
// compressed W (bitmap + packed f16 values), W never written to HBM.
//
// The reference has no consumer (compute is a constant, sim.hpp:30,227); the
// decompress it feeds is codec.hpp:157-166.  Decompress + GEMV moves
// 1/8 + (1-s)*2 (read) + 2 (write) + 2 (re-read) B per weight; fused moves
// only 1/8 + (1-s)*2 -- 1.125 B at 50 % instead of 5.125.  At that traffic the
// kernel has to expand ~5.8 G weights/ms to stay HBM-bound, so the design is
// about instructions and shared-memory wavefronts per weight:
//
//  * work item t = 8 consecutive 1024-element sub-tiles [8t, 8t+8) of the
//    flattened matrix (the RankIndex chunks): one contiguous bitmap kilobyte
//    and one contiguous packed-value window, so one producer warp moves an
//    item with two 1-D TMA bulk copies (bitmap, values) into a 4-stage smem
//    ring (cp.async.bulk + mbarrier complete_tx).  The item's nine index
//    entries are fetched 32 items ahead (one per lane), validated (monotone,
//    within [0, nnz], at most 1024 apart) and written to the stage as 32-bit
//    offsets relative to the value window;
//  * consumer warp w takes sub-tile 8t + w, i.e. column segment
//    (8t + w) % segs.  A CTA walks items t0, t0 + segs, t0 + 2 segs, ..
//    (the same 8 segments one 8-row band further down each time), so every
//    warp's x segment (1024 f16 = 16 registers per lane) stays in registers
//    for the whole run;
//  * lane l expands bitmap bytes l, l+32, .. of the sub-tile (8 weights, two
//    nibbles each; ENDOR_GV_BYTE_LANES=0 selects nibble lanes, conflict-free
//    LDS but twice the shuffles -- measured slower): PRMT selector gathers
//    (gather.cuh) place the packed values and FHFMA (fp32 += f16*f16, one
//    instruction per weight, predicated for unset slots) accumulates; the
//    fp32 partial of each sub-tile goes to the workspace and a second tiny
//    kernel sums each row's partials in a fixed order (deterministic, no
//    atomics).  ~300 warp-instructions per 1024 weights: issue-bound (ncu
//    71 % issue, 78 % L1), independent of the density.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "gather.cuh"
#include "kernels.h"

namespace endor_b200 {

constexpr int kGvWarps = 8;                       // sub-tiles per item = consumer warps
constexpr int kGvThreads = (kGvWarps + 1) * 32;   // + 1 producer warp
#ifndef ENDOR_GV_STAGES
#define ENDOR_GV_STAGES 4
#endif
constexpr int kGvStages = ENDOR_GV_STAGES;
constexpr uint64_t kGvSparseDensity10 = 2;  // set-bit consumer at density <= 0.2 (tools/fused_sweep.py)
// lane granularity of the gather: 1 = byte lanes (two nibbles per step, one
// shuffle pair per 8 weights), 0 = nibble lanes (conflict-free LDS)
#ifndef ENDOR_GV_BYTE_LANES
#define ENDOR_GV_BYTE_LANES 1
#endif
constexpr uint32_t kGvBm = 0;                                  // 8 x 128-byte bitmap slices
constexpr uint32_t kGvMeta = kGvWarps * 128;                   // 9 u32 sub-tile starts relative to the
                                                               // window, then the window's byte offset
constexpr uint32_t kGvVals = kGvMeta + 48;                     // packed-value window
constexpr uint32_t kGvStage = kGvVals + kGvWarps * kSubElems * 2 + 32 + 64;  // + alignment slack + over-read pad
// SPARSE consumer (density <= 0.2): each lane walks the set bits of its own bitmap
// word -- cost per set value, not per slot.  x (1024 f16 per warp) lives in
// shared memory transposed (column 32 l + b at b * 32 + l: at most 2-way bank
// conflicts for any per-lane bit), so one stage fewer keeps 3 CTAs per SM.
template <bool SPARSE>
constexpr int gv_stages() { return SPARSE ? kGvStages - 1 : kGvStages; }
template <bool SPARSE>
constexpr uint32_t gv_smem() { return 256 + gv_stages<SPARSE>() * kGvStage + (SPARSE ? kGvWarps * kSubElems * 2 : 0); }

// inclusive warp prefix sum: shfl.up's in-range predicate guards each add
__device__ __forceinline__ uint32_t warp_incl_scan_p(uint32_t v) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1)
        asm("{\n\t.reg .u32 u;\n\t.reg .pred p;\n\t"
            "shfl.sync.up.b32 u|p, %0, %1, 0, 0xffffffff;\n\t"
            "@p add.u32 %0, %0, u;\n\t}"
            : "+r"(v) : "r"(d));
    return v;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// sel = g_lut16[nib] with the address formed as base + 4*nib (one LEA)
__device__ __forceinline__ uint32_t lut_sel(uint32_t lut_base, uint32_t nib) {
    uint32_t v;
    asm("{\n\t.reg .u32 t;\n\tmad.lo.u32 t, %1, 4, %2;\n\tld.shared.u32 %0, [t];\n\t}"
        : "=r"(v) : "r"(nib), "r"(lut_base));
    return v;
}

// {sel0, sel1} per nibble in one LDS.64 (ENDOR_GV_LUT64): no shift for the slot-2/3 selector
#ifndef ENDOR_GV_LUT64
#define ENDOR_GV_LUT64 1  // measured 0.7 % faster than LDS.32 + shift (profiles/r02/fused_gemv_hmma_experiment.txt)
#endif
__shared__ uint2 g_lut_gv[16];
__device__ __forceinline__ uint2 lut_gv(uint32_t lut_base, uint32_t nib) {
    uint2 v;
    asm("{\n\t.reg .u32 t;\n\tmad.lo.u32 t, %2, 8, %3;\n\tld.shared.v2.u32 {%0, %1}, [t];\n\t}"
        : "=r"(v.x), "=r"(v.y) : "r"(nib), "r"(lut_base));
    return v;
}

// acc += w.lo * x.lo if (nib & LO), + w.hi * x.hi if (nib & HI): unset slots
// hold arbitrary bytes and are skipped instead of zeroed (fp32 += f16 * f16)
template <uint32_t LO, uint32_t HI>
__device__ __forceinline__ float fma_f16x2_if(uint32_t w, uint32_t x, float acc, uint32_t nib) {
    asm("{\n\t.reg .b16 wl, wh, xl, xh;\n\t.reg .pred p;\n\t.reg .u32 t;\n\t"
        "mov.b32 {wl, wh}, %1;\n\t"
        "mov.b32 {xl, xh}, %2;\n\t"
        "and.b32 t, %3, %4;\n\tsetp.ne.u32 p, t, 0;\n\t"
        "@p fma.rn.f32.f16 %0, wl, xl, %0;\n\t"
        "and.b32 t, %3, %5;\n\tsetp.ne.u32 p, t, 0;\n\t"
        "@p fma.rn.f32.f16 %0, wh, xh, %0;\n\t}"
        : "+f"(acc) : "r"(w), "r"(x), "r"(nib), "n"(LO), "n"(HI));
    return acc;
}

// Item walk.  Per tensor: nsub sub-tiles, T = ceil(nsub / 8) items, segs
// item columns; column c holds items c, c + segs, c + 2 segs, .. (its first
// (T mod segs) columns one more than the rest).  The CTA's linear item range
// runs column-major, tensor after tensor.
struct ItemCursor {
    int ti;
    uint64_t segs, nitems, q, r0;  // per tensor: T, T / segs, T % segs
    uint64_t col, j, clen;         // current column, index in it, column length
    __device__ void load(const Batch& b) {
        const BatchTensor& T = b.t[ti];
        segs = T.cols / kSubElems;
        nitems = ceil_div(T.n / kSubElems, kGvWarps);
        q = nitems / segs;
        r0 = nitems - q * segs;
    }
    __device__ void init(const Batch& b, uint64_t u) {
        ti = 0;
        while (ti + 1 < b.count && u >= b.t[ti + 1].item0) ++ti;
        load(b);
        uint64_t lu = u - b.t[ti].item0;
        if (lu < r0 * (q + 1)) {
            col = lu / (q + 1);
            j = lu - col * (q + 1);
        } else {
            lu -= r0 * (q + 1);
            col = r0 + lu / q;
            j = lu - (col - r0) * q;
        }
        clen = q + (col < r0);
    }
    __device__ void next(const Batch& b) {
        if (++j < clen) return;
        j = 0;
        if (++col == segs) {
            if (ti + 1 >= b.count) return;  // past the batch: callers check the item bound
            col = 0;
            ++ti;
            load(b);
        }
        clen = q + (col < r0);
    }
    __device__ uint64_t item() const { return col + j * segs; }
};

#ifndef ENDOR_GV_MINB
#define ENDOR_GV_MINB 3  // CTAs per SM the register budget is sized for
#endif
template <bool SPARSE>
__global__ void __launch_bounds__(kGvThreads, ENDOR_GV_MINB) gemv_fused_kernel(const __grid_constant__ Batch b, uint64_t nitems) {
    constexpr int kGvStages = gv_stages<SPARSE>();
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sbase = smem_u32(smem);
    const uint32_t full0 = sbase, empty0 = sbase + 8 * kGvStages;
    const uint32_t st0 = sbase + 256;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    init_luts(tid);
    if (ENDOR_GV_LUT64 && tid < 16) g_lut_gv[tid] = make_uint2(g_lut16[tid] & 0xFFFFu, g_lut16[tid] >> 16);
    if (tid == 0) {
        for (int s = 0; s < kGvStages; ++s) {
            mbar_init(full0 + 8 * s, 2);          // producer: expect_tx arrive + fix-up arrive
            mbar_init(empty0 + 8 * s, kGvWarps);  // one arrive per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_wait();
    if (cta_error_latched(b.hdr)) return;  // a latched error: write nothing (+ publishes the prologue)
    pdl_launch_dependents();
    if (warp == kGvWarps) {
        // check_index's tail test (codec.hpp:177-183), tensor t on CTA grid - 1 - t
        // (one test per CTA instead of a batch's worth serially on CTA 0)
        for (int t = int(gridDim.x - 1 - blockIdx.x); t < b.count; t += int(gridDim.x)) {
            const BatchTensor& T = b.t[t];
            const uint64_t last = T.n / kSubElems - 1;  // n % 1024 == 0 here
            const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(T.bitmap) + last * 32 + lane);
            const uint32_t tail = __reduce_add_sync(0xffffffffu, __popc(v));
            if (lane == 0 && T.idx[last] + tail != T.nnz) latch_status(b.hdr, ENDOR_ERR_CORRUPTION);
        }
    }
    // this CTA's contiguous range of the column-major item order
    const uint64_t u0 = nitems * blockIdx.x / gridDim.x, u1 = nitems * (blockIdx.x + 1) / gridDim.x;
    if (u0 >= u1) return;
    const uint32_t m = uint32_t(u1 - u0);

    if (warp == kGvWarps) {
        // ================= producer warp =================
        // lane l holds item i + l of the current / next 32-item group: its
        // nine sub-tile starts idx[8t .. 8t+8] (nnz past the end), fetched one
        // group ahead and validated here -- monotone and within [0, nnz] --
        // so consumers work with 32-bit offsets relative to the window
        unsigned long long ce[kGvWarps + 1], ne[kGvWarps + 1];
        uint64_t ct = 0, nt = 0;
        int cti = 0, nti = 0;
        auto fetch = [&](uint32_t base, unsigned long long* e, uint64_t& wt, int& wti) {
            if (base + lane >= m) return;
            ItemCursor c;
            c.init(b, u0 + base + lane);
            const BatchTensor& T = b.t[c.ti];
            const uint64_t t = c.item(), nsub = T.n / kSubElems;
#pragma unroll
            for (int q = 0; q <= kGvWarps; ++q) e[q] = 8 * t + q < nsub ? T.idx[8 * t + q] : T.nnz;
            wt = t;
            wti = c.ti;
        };
        auto validate = [&](unsigned long long* e, int wti) {  // clamp + latch (memory safety)
            const unsigned long long nnz = b.t[wti].nnz;
            bool bad = false;
            unsigned long long lo = 0;
#pragma unroll
            for (int q = 0; q <= kGvWarps; ++q) {
                unsigned long long v = e[q] < lo ? lo : (e[q] > nnz ? nnz : e[q]);
                if (q > 0 && v - e[0] > uint64_t(q) * kSubElems) v = e[0] + uint64_t(q) * kSubElems;
                bad |= v != e[q];
                e[q] = lo = v;
            }
            if (bad) latch_status(b.hdr, ENDOR_ERR_CORRUPTION);
        };
        fetch(0, ce, ct, cti);
        fetch(32, ne, nt, nti);
        if (lane < int(m)) validate(ce, cti);
        for (uint32_t i = 0; i < m; ++i) {
            if (i % 32 == 0 && i > 0) {
#pragma unroll
                for (int q = 0; q <= kGvWarps; ++q) ce[q] = ne[q];
                ct = nt;
                cti = nti;
                if (i + lane < m) validate(ce, cti);
                fetch(i + 32, ne, nt, nti);
            }
            const int s = int(i % kGvStages);
            const uint32_t stg = st0 + s * kGvStage, full = full0 + 8 * s;
            const int src = int(i & 31);
            const unsigned long long s0 = __shfl_sync(0xffffffffu, ce[0], src);
            const unsigned long long s1 = __shfl_sync(0xffffffffu, ce[kGvWarps], src);
            const uint64_t t = __shfl_sync(0xffffffffu, ct, src);
            const BatchTensor& T = b.t[__shfl_sync(0xffffffffu, cti, src)];
            const uint32_t nk = uint32_t(umin64(kGvWarps, T.n / kSubElems - 8 * t));  // sub-tiles in this item
            const uintptr_t vlo = reinterpret_cast<uintptr_t>(T.values), vhi = vlo + T.nnz * 2;
            const uintptr_t vlo16 = (vlo + 15) & ~uintptr_t(15), vhi16 = vhi & ~uintptr_t(15);
            const uintptr_t ws = vlo + s0 * 2, we = vlo + s1 * 2;
            const uintptr_t as = ws & ~uintptr_t(15), ae = (we + 15) & ~uintptr_t(15);
            const uintptr_t bs = as > vlo16 ? as : vlo16, be = ae < vhi16 ? ae : vhi16;
            const uint32_t vbulk = be > bs ? uint32_t(be - bs) : 0u;
            if (i >= uint32_t(kGvStages)) mbar_wait(empty0 + 8 * s, ((i / kGvStages) - 1) & 1);
            if (lane == 0) {
                mbar_arrive_expect_tx(full, nk * 128 + vbulk);
                bulk_g2s(stg + kGvBm, T.bitmap + t * (kGvWarps * 128), nk * 128, full);
                if (vbulk) bulk_g2s(stg + kGvVals + uint32_t(bs - as), reinterpret_cast<const void*>(bs), vbulk, full);
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(stg + kGvMeta + 36), "r"(uint32_t(ws - as)) : "memory");
            }
            if (lane == src) {  // the item's owner lane: sub-tile starts relative to the window
                uint32_t r[kGvWarps + 1];
#pragma unroll
                for (int q = 0; q <= kGvWarps; ++q) r[q] = uint32_t(ce[q] - ce[0]);
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(stg + kGvMeta), "r"(r[0]), "r"(r[1]),
                             "r"(r[2]), "r"(r[3]) : "memory");
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(stg + kGvMeta + 16), "r"(r[4]),
                             "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(stg + kGvMeta + 32), "r"(r[8]) : "memory");
            }
            if (bs > ws || be < we) {  // edge bytes of the buffer the bulk copy cannot move
                const uintptr_t e0 = vbulk ? bs : we, e1 = vbulk ? be : we;
                for (uintptr_t p = ws + lane; p < e0 && p < we; p += 32)
                    sts8(stg + kGvVals + uint32_t(p - as), *reinterpret_cast<const uint8_t*>(p));
                for (uintptr_t p = (e1 > ws ? e1 : ws) + lane; p < we; p += 32)
                    sts8(stg + kGvVals + uint32_t(p - as), *reinterpret_cast<const uint8_t*>(p));
                fence_proxy_async_smem();  // st.shared edges vs the TMA that later reuses the stage
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(full);
        }
        return;
    }

    // ================= consumer warps: sub-tile 8t + warp of every item =================
    ItemCursor cur;
    cur.init(b, u0);
    uint32_t xrun = ~0u, run = 0;     // column run id: x reloads only when it changes
    uint64_t k = cur.item() * kGvWarps + warp, nsub = b.t[cur.ti].n / kSubElems;
    uint32_t xr[16];  // x[4n .. 4n+3] for this lane's nibbles n = lane + 32 q of the segment
#if ENDOR_GV_BYTE_LANES
    const uint32_t nsh = (lane & 3) * 8, lowm = (1u << nsh) - 1u;  // lane's byte inside its word
#else
    const uint32_t nsh = (lane & 7) * 4, lowm = (1u << nsh) - 1u;  // lane's nibble inside its word
#endif
    const uint32_t lut = smem_u32(g_lut16);
    const BatchTensor* T = &b.t[cur.ti];
    for (uint32_t i = 0; i < m; ++i) {
        const bool ok = k < nsub;
        if (SPARSE && ok && run != xrun) {  // x segment -> this warp's smem, transposed
            const uint32_t xs = st0 + kGvStages * kGvStage + warp * (kSubElems * 2);
            const uint4* src = static_cast<const uint4*>(T->x) + (k % cur.segs) * (kSubElems / 8) + lane * 4;
            __syncwarp();  // the previous run's reads are done
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 v = __ldg(src + q);
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int h = 0; h < 8; ++h) {  // column 32 lane + 8 q + h
                    const uint32_t bcol = 8 * q + h;
                    asm volatile("st.shared.u16 [%0], %1;" ::"r"(xs + 2 * (bcol * 32 + lane)),
                                 "h"(uint16_t(w4[h >> 1] >> (16 * (h & 1)))) : "memory");
                }
            }
            __syncwarp();
            xrun = run;
        }
        if (!SPARSE && ok && run != xrun) {  // x stays in registers along a column
#if ENDOR_GV_BYTE_LANES
            const uint4* xs = static_cast<const uint4*>(T->x) + (k % cur.segs) * (kSubElems / 8);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 v = __ldg(xs + 32 * q + lane);
                xr[4 * q] = v.x;
                xr[4 * q + 1] = v.y;
                xr[4 * q + 2] = v.z;
                xr[4 * q + 3] = v.w;
            }
#else
            const uint2* xs = static_cast<const uint2*>(T->x) + (k % cur.segs) * (kSubElems / 4);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint2 v = __ldg(xs + 32 * q + lane);
                xr[2 * q] = v.x;
                xr[2 * q + 1] = v.y;
            }
#endif
            xrun = run;
        }
        const int s = int(i % kGvStages);
        const uint32_t stg = st0 + s * kGvStage;
        mbar_wait(full0 + 8 * s, (i / kGvStages) & 1);
        if (ok) {
            const uint32_t off = lds32(stg + kGvMeta + 36);
            const uint32_t r0 = lds32(stg + kGvMeta + 4 * warp), r1 = lds32(stg + kGvMeta + 4 + 4 * warp);
            uint32_t word = lds32(stg + kGvBm + warp * 128 + lane * 4);
            const uint32_t pc = __popc(word);
            const uint32_t incl = warp_incl_scan_p(pc);
            const uint32_t wtotal = __shfl_sync(0xffffffffu, incl, 31);
            // byte address of word l's first packed value
            uint32_t wbase = stg + kGvVals + off + 2 * (r0 + incl - pc);
            if (wtotal != r1 - r0) {  // popcount disagrees with the index: latch, stay in bounds
                if (lane == 0) latch_status(b.hdr, ENDOR_ERR_CORRUPTION);
                word = 0;
                wbase = stg + kGvVals;
            }
            float acc0 = 0.f, acc1 = 0.f;
            if constexpr (SPARSE) {
                // lane l: the set bits of word l, values from its exclusive rank on
                const uint32_t xs = st0 + kGvStages * kGvStage + warp * (kSubElems * 2) + 2 * lane;
                uint32_t a = wbase;  // this word's first packed value
                uint32_t w = word;
                if ((a & 1) == 0) {
                    while (w) {
                        const uint32_t bit = __ffs(w) - 1;
                        w &= w - 1;
                        uint16_t v, xv;
                        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
                        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(xv) : "r"(xs + 64 * bit));
                        asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc0) : "h"(v), "h"(xv));
                        a += 2;
                    }
                } else {  // an odd values buffer (any alignment is allowed): two byte loads
                    while (w) {
                        const uint32_t bit = __ffs(w) - 1;
                        w &= w - 1;
                        uint16_t v0, v1, xv;
                        asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v0) : "r"(a));
                        asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v1) : "r"(a + 1));
                        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(xv) : "r"(xs + 64 * bit));
                        const uint16_t v = uint16_t(v0 | (v1 << 8));
                        asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc0) : "h"(v), "h"(xv));
                        a += 2;
                    }
                }
            } else {
#if ENDOR_GV_BYTE_LANES
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int src = 8 * q + (lane >> 2);  // word of byte lane + 32 q
                const uint32_t wd = __shfl_sync(0xffffffffu, word, src);
                const uint32_t a0 = __shfl_sync(0xffffffffu, wbase, src) + 2 * __popc(wd & lowm);
                const uint32_t byte = (wd >> nsh) & 0xFFu;
                const uint32_t n0 = byte & 15u, n1 = byte >> 4;
                const uint32_t a1 = a0 + 2 * __popc(n0);
                // nibble 0 at a0, nibble 1 at a1: 4 packed values each -> 8 slots
#if ENDOR_GV_LUT64
                const uint2 e0 = lut_gv(smem_u32(g_lut_gv), n0), e1 = lut_gv(smem_u32(g_lut_gv), n1);
                const uint32_t s0 = e0.x, s1 = e1.x, s0h = e0.y, s1h = e1.y;
#else
                const uint32_t s0 = lut_sel(lut, n0), s1 = lut_sel(lut, n1);
                const uint32_t s0h = s0 >> 16, s1h = s1 >> 16;
#endif
                const uint32_t l0 = a0 & ~3u, h0 = a0 << 3, l1 = a1 & ~3u, h1 = a1 << 3;
                const uint32_t u0 = lds32(l0), u1 = lds32(l0 + 4), u2 = lds32(l0 + 8);
                const uint32_t v0 = lds32(l1), v1 = lds32(l1 + 4), v2 = lds32(l1 + 8);
                const uint32_t x0 = __funnelshift_r(u0, u1, h0), y0 = __funnelshift_r(u1, u2, h0);
                const uint32_t x1 = __funnelshift_r(v0, v1, h1), y1 = __funnelshift_r(v1, v2, h1);
                acc0 = fma_f16x2(prmt(x0, 0u, s0), xr[4 * q], acc0);
                acc1 = fma_f16x2_if<0x4u, 0x8u>(prmt(x0, y0, s0h), xr[4 * q + 1], acc1, byte);
                acc0 = fma_f16x2(prmt(x1, 0u, s1), xr[4 * q + 2], acc0);
                acc1 = fma_f16x2_if<0x40u, 0x80u>(prmt(x1, y1, s1h), xr[4 * q + 3], acc1, byte);
            }
#else
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int src = 4 * q + (lane >> 3);  // word of nibble lane + 32 q
                const uint32_t wd = __shfl_sync(0xffffffffu, word, src);
                const uint32_t a = __shfl_sync(0xffffffffu, wbase, src) + 2 * __popc(wd & lowm);
                const uint32_t nib = (wd >> nsh) & 15u;
                // 4 packed values at byte address a (2-aligned) -> the nibble's slots
                const uint32_t sel = lut_sel(lut, nib);
                const uint32_t al = a & ~3u, sh = a << 3;
                const uint32_t w0 = lds32(al), w1 = lds32(al + 4), w2 = lds32(al + 8);
                const uint32_t x = __funnelshift_r(w0, w1, sh), y = __funnelshift_r(w1, w2, sh);
                acc0 = fma_f16x2(prmt(x, 0u, sel), xr[2 * q], acc0);  // slots 0, 1 (unset -> +0)
                acc1 = fma_f16x2_if<4u, 8u>(prmt(x, y, sel >> 16), xr[2 * q + 1], acc1, nib);  // slots 2, 3
            }
#endif
            }
            float a = acc0 + acc1;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) a += __shfl_xor_sync(0xffffffffu, a, d);
            if (lane == 0) T->part[k] = a;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * s);
        // next item: same column -> 8 rows' worth of sub-tiles further on
        const int ti = cur.ti;
        const uint64_t col = cur.col;
        cur.next(b);
        if (cur.ti != ti || cur.col != col) {
            ++run;
            T = &b.t[cur.ti];
            nsub = T->n / kSubElems;
            k = cur.item() * kGvWarps + warp;
        } else {
            k += cur.segs * kGvWarps;
        }
    }
}

// count_kernel's two-level offsets -> a flat 1024-chunk RankIndex, in place
// (tsub[k] += blk[k / subs_per_count_cta]), for the tensors without a
// caller index; the fused kernel then reads one table.
struct FlattenBatch {
    unsigned long long* tsub[kMaxBatch];
    const unsigned long long* blk[kMaxBatch];
    uint64_t spc[kMaxBatch];
    uint64_t sub0[kMaxBatch + 1];
    int count;
};

__global__ void __launch_bounds__(256) flatten_kernel(const __grid_constant__ FlattenBatch f) {
    pdl_wait();
    pdl_launch_dependents();
    const uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= f.sub0[f.count]) return;
    int k = 0;
    while (g >= f.sub0[k + 1]) ++k;
    const uint64_t j = g - f.sub0[k];
    f.tsub[k][j] += f.blk[k][j / f.spc[k]];
}

cudaError_t launch_flatten(unsigned long long* tsub, const unsigned long long* blk, uint64_t spc, uint64_t count,
                           cudaStream_t s) {
    if (!count) return cudaSuccess;
    FlattenBatch f{};
    f.tsub[0] = tsub;
    f.blk[0] = blk;
    f.spc[0] = spc;
    f.sub0[0] = 0;
    f.sub0[1] = count;
    f.count = 1;
    return launch_pdl(flatten_kernel, dim3(unsigned(ceil_div(count, 256))), dim3(256), 0, s, f);
}

cudaError_t launch_gemv_fused(Batch& b, cudaStream_t s) {
    FlattenBatch f{};
    uint64_t nflat = 0;
    for (int k = 0; k < b.count; ++k) {
        BatchTensor& T = b.t[k];
        if (T.idx) continue;
        f.tsub[f.count] = b.tsub + T.sub0;
        f.blk[f.count] = b.blk + T.blk0;
        f.spc[f.count] = uint64_t(kCountSubs) * T.cbpc;
        f.sub0[f.count] = nflat;
        nflat += T.n / kSubElems;
        T.idx = b.tsub + T.sub0;  // absolute offsets after the flatten pass
        ++f.count;
    }
    f.sub0[f.count] = nflat;
    if (nflat) {
        cudaError_t e = launch_pdl(flatten_kernel, dim3(unsigned(ceil_div(nflat, 256))), dim3(256), 0, s, f);
        if (e != cudaSuccess) return e;
    }
    int blocks_per_sm = 1, sms = 148;
    // per-batch consumer choice by density (ENDOR_GV_SPARSE=0/1 forces one)
    uint64_t n_all = 0, nnz_all = 0;
    for (int k = 0; k < b.count; ++k) {
        n_all += b.t[k].n;
        nnz_all += b.t[k].nnz;
    }
    static const int env_sparse = [] {
        const char* e = getenv("ENDOR_GV_SPARSE");
        return e ? atoi(e) : -1;
    }();
    const bool sparse = env_sparse >= 0 ? env_sparse != 0 : nnz_all * 10 <= n_all * kGvSparseDensity10;
    const void* fn = sparse ? reinterpret_cast<const void*>(gemv_fused_kernel<true>)
                            : reinterpret_cast<const void*>(gemv_fused_kernel<false>);
    const uint32_t smem = sparse ? gv_smem<true>() : gv_smem<false>();
    cudaError_t e = kernel_slots(fn, kGvThreads, smem, &blocks_per_sm, &sms);
    if (e != cudaSuccess) return e;
    uint64_t items = 0;
    for (int k = 0; k < b.count; ++k) {
        BatchTensor& T = b.t[k];
        T.item0 = items;
        items += ceil_div(T.n / kSubElems, kGvWarps);
    }
    const uint64_t grid = umin64(items, uint64_t(blocks_per_sm) * sms);
    if (grid == 0) return cudaSuccess;
    if (sparse) return launch_pdl(gemv_fused_kernel<true>, dim3(unsigned(grid)), dim3(kGvThreads), smem, s, b, items);
    return launch_pdl(gemv_fused_kernel<false>, dim3(unsigned(grid)), dim3(kGvThreads), smem, s, b, items);
}

// y[r] = sum over the row's segment partials in segment order (deterministic)
struct ReduceBatch {
    const float* part[kMaxBatch];
    float* y32[kMaxBatch];
    __half* y16[kMaxBatch];
    uint64_t row0[kMaxBatch + 1];
    uint32_t segs[kMaxBatch];
    int count;
};

__global__ void __launch_bounds__(256) row_reduce_kernel(const __grid_constant__ ReduceBatch rb) {
    pdl_wait();
    pdl_launch_dependents();
    const uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= rb.row0[rb.count]) return;
    int k = 0;
    while (g >= rb.row0[k + 1]) ++k;
    const uint64_t r = g - rb.row0[k];
    const float* p = rb.part[k] + r * rb.segs[k];
    float acc = 0.f;
    for (uint32_t j = 0; j < rb.segs[k]; ++j) acc += p[j];
    if (rb.y32[k]) rb.y32[k][r] = acc;
    if (rb.y16[k]) rb.y16[k][r] = __float2half_rn(acc);
}

cudaError_t launch_row_reduce_batch(const Batch& b, float* const* y32, void* const* y16, cudaStream_t s) {
    ReduceBatch rb{};
    rb.count = b.count;
    uint64_t rows = 0;
    for (int k = 0; k < b.count; ++k) {
        rb.part[k] = b.t[k].part;
        rb.y32[k] = y32 ? y32[k] : nullptr;
        rb.y16[k] = y16 ? static_cast<__half*>(y16[k]) : nullptr;
        rb.segs[k] = uint32_t(b.t[k].cols / kSubElems);
        rb.row0[k] = rows;
        rows += b.t[k].n / b.t[k].cols;
    }
    rb.row0[b.count] = rows;
    if (rows == 0) return cudaSuccess;
    return launch_pdl(row_reduce_kernel, dim3(unsigned(ceil_div(rows, 256))), dim3(256), 0, s, rb);
}

}  // namespace endor_b200
