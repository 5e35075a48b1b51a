// decompress.cu -- sm_100a kernels for the Endor hot path.
//
//   scan_kernel    per-range popcount + decoupled look-back exclusive scan.
//                  Produces the per-tile value offsets the expand kernel
//                  needs (the device RankIndex), writes/verifies a caller's
//                  RankIndex at its chunk size (build_rank_index,
//                  bitmap.hpp:117-132; check_index, codec.hpp:170-184),
//                  and checks popcount == nnz (codec.hpp:158-160).
//   expand_kernel  one CTA per 8192-element tile: bitmap words -> block scan
//                  of __popc -> values window staged into shared memory with
//                  16-byte loads -> 16-byte coalesced dense stores.  This is
//                  detail::scatter_range (codec.hpp:132-152) with the serial
//                  value cursor `v` replaced by prefix sums.
//
// Both are HBM-bound integer/byte kernels (no tensor cores: there is no
// GEMM-shaped work in a bitmap expansion).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace endor_b200 {

__global__ void __launch_bounds__(kScanThreads) scan_kernel(ScanArgs a) {
    __shared__ uint32_t s_ticket;
    __shared__ unsigned long long s_warp_tot[kScanThreads / 32];
    __shared__ unsigned long long s_excl;
    __shared__ int s_last;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_ticket = uint32_t(atomicAdd(&a.hdr->ticket, 1ull));
    __syncthreads();
    const uint32_t blk = s_ticket;  // tickets are handed out in launch order

    const uint64_t wbase = a.e0 / 32;                     // first word of the range
    const uint64_t wend = (a.e1 + 31) / 32;               // one past the last word
    const uint64_t seg = uint64_t(blk) * kScanBlockWords + uint64_t(warp) * kScanWarpWords;

    // ---- phase 1: coalesced word loads + per-lane popcounts ----------------
    uint32_t w[kScanWordsPerLane];
    uint32_t lane_cnt = 0;
#pragma unroll
    for (int j = 0; j < kScanWordsPerLane; ++j) {
        const uint64_t rel = seg + uint64_t(j) * 32 + lane;  // word index relative to e0
        const uint64_t wi = wbase + rel;
        uint32_t v = 0;
        if (wi < wend) {
            v = load_word32(a.bitmap, wi, a.nbytes);
            const uint64_t bit0 = wi * 32;
            if (bit0 + 32 > a.e1) {
                const uint32_t keep = uint32_t(a.e1 - bit0);  // 1..31
                // Padding bits of the final byte must be zero (bitmap.hpp:78-84).
                if (a.e1 == a.n && (a.n & 7)) {
                    const uint64_t pad_end = ((a.n + 7) & ~7ull) - bit0;  // bits < pad_end loaded
                    const uint32_t padmask = (pad_end >= 32 ? 0xffffffffu : ((1u << pad_end) - 1u)) &
                                             ~((1u << keep) - 1u);
                    if (v & padmask) latch_status(a.hdr, ENDOR_ERR_CORRUPTION);
                }
                v &= (1u << keep) - 1u;
            }
        }
        w[j] = v;
        lane_cnt += __popc(v);
    }
    uint32_t warp_cnt = lane_cnt;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) warp_cnt += __shfl_xor_sync(0xffffffffu, warp_cnt, d);
    if (lane == 0) s_warp_tot[warp] = warp_cnt;
    __syncthreads();

    // ---- phase 2: block aggregate + decoupled look-back ----------------------
    if (tid == 0) {
        unsigned long long agg = 0;
        for (int i = 0; i < kScanThreads / 32; ++i) {
            const unsigned long long t = s_warp_tot[i];
            s_warp_tot[i] = agg;  // now the warp's exclusive offset within the block
            agg += t;
        }
        unsigned long long base = a.p0_ptr ? *a.p0_ptr : a.p0;
        unsigned long long excl = 0;
        if (blk == 0) {
            lb_store(&a.lookback[0], kLbPrefix | (agg & kLbValue));
        } else {
            lb_store(&a.lookback[blk], kLbAgg | (agg & kLbValue));
            for (int64_t j = int64_t(blk) - 1; j >= 0;) {
                const unsigned long long s = lb_load(&a.lookback[j]);
                const unsigned long long f = s & ~kLbValue;
                if (f == 0) continue;  // predecessor has not published yet: spin
                excl += s & kLbValue;
                if (f == kLbPrefix) break;
                --j;
            }
            lb_store(&a.lookback[blk], kLbPrefix | ((excl + agg) & kLbValue));
        }
        s_excl = base + excl;
        if (blk == a.nblocks - 1) {
            const unsigned long long total = base + excl + agg;
            if (a.total_out) *a.total_out = total;
            a.hdr->total = total;
            if (a.check_total && total != a.expect_total) latch_status(a.hdr, ENDOR_ERR_CORRUPTION);
        }
    }
    __syncthreads();

    // ---- phase 3: per-word exclusive offsets at tile / chunk starts -----------
    unsigned long long running = s_excl + s_warp_tot[warp];
    const bool want_chunks = a.cs != 0 && (a.idx_out || a.idx_in);
#pragma unroll
    for (int j = 0; j < kScanWordsPerLane; ++j) {
        const uint32_t pc = __popc(w[j]);
        const uint32_t incl = warp_incl_scan(pc, lane);
        const unsigned long long excl = running + (incl - pc);
        const uint64_t rel = seg + uint64_t(j) * 32 + lane;
        const uint64_t wi = wbase + rel;
        if (wi < wend) {
            if (a.tprefix && (rel % kTileWords) == 0) a.tprefix[rel / kTileWords] = excl;
            if (want_chunks) {
                const uint64_t bit = wi * 32;
                if ((bit & (a.cs - 1)) == 0) {
                    const uint64_t k = bit / a.cs;
                    if (a.idx_out) a.idx_out[k] = excl;
                    else if (a.idx_in[k] != excl) latch_status(a.hdr, ENDOR_ERR_CORRUPTION);
                }
            }
        }
        running += __shfl_sync(0xffffffffu, incl, 31);
    }

    // ---- self-reset of the look-back state (workspace stays zeroed) -----------
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const unsigned long long d = atomicAdd(&a.hdr->done, 1ull);
        s_last = (d == a.nblocks - 1);
    }
    __syncthreads();
    if (s_last) {
        for (uint32_t i = tid; i < a.nblocks; i += kScanThreads) a.lookback[i] = 0;
        if (tid == 0) {
            a.hdr->ticket = 0;
            a.hdr->done = 0;
        }
    }
}

// ---------------------------------------------------------------------------
// expand
// ---------------------------------------------------------------------------
// Gather one 16-byte output chunk: element k of the chunk takes the next
// packed value when bit k of m is set, else +0 (codec.hpp:136,144-149).
template <int EB, bool ALIGNED>
__device__ __forceinline__ uint4 gather_chunk(uint32_t m, uint32_t p, const uint8_t* s) {
    uint32_t o[4] = {0u, 0u, 0u, 0u};
    if constexpr (EB == 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (m & (1u << k)) {
                uint32_t v;
                if constexpr (ALIGNED) v = *reinterpret_cast<const uint16_t*>(s + p);
                else v = uint32_t(s[p]) | (uint32_t(s[p + 1]) << 8);
                o[k >> 1] |= v << ((k & 1) * 16);
                p += 2;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (m & (1u << k)) {
                o[k >> 2] |= uint32_t(s[p]) << ((k & 3) * 8);
                p += 1;
            }
        }
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

template <int EB>
__global__ void __launch_bounds__(kExpandThreads, 8) expand_kernel(ExpandArgs a) {
    constexpr int EPC = 16 / EB;  // elements per 16-byte chunk
    constexpr uint32_t CMASK = (EPC == 32) ? 0xffffffffu : ((1u << EPC) - 1u);
    __shared__ uint32_t s_word[kTileWords];
    __shared__ uint32_t s_wpre[kTileWords];
    __shared__ uint32_t s_warp[kExpandThreads / 32];
    __shared__ __align__(16) uint8_t s_vals[kTileElems * EB + 32];

    if (read_status(a.hdr)) return;  // a latched error: write nothing
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t t0 = a.e0 + uint64_t(blockIdx.x) * kTileElems;
    const uint64_t tend = min(a.e1, t0 + kTileElems);
    const uint32_t count = uint32_t(tend - t0);

    // bitmap word for this thread (32 elements), bits past the range masked
    uint32_t wv = 0;
    if (uint32_t(tid) * 32 < count) {
        wv = load_word32(a.bitmap, t0 / 32 + tid, a.nbytes);
        const uint32_t rem = count - uint32_t(tid) * 32;
        if (rem < 32) wv &= (1u << rem) - 1u;
    }
    const uint32_t pc = __popc(wv);
    const uint32_t incl = warp_incl_scan(pc, lane);
    if (lane == 31) s_warp[warp] = incl;
    s_word[tid] = wv;
    __syncthreads();
    uint32_t wexcl = 0, total = 0;
#pragma unroll
    for (int i = 0; i < kExpandThreads / 32; ++i) {
        const uint32_t t = s_warp[i];
        wexcl += (i < warp) ? t : 0u;
        total += t;
    }
    s_wpre[tid] = wexcl + incl - pc;

    // values window [vbase, vbase+total) -> shared memory, aligned superset
    const uint64_t vbase = a.tprefix[blockIdx.x];
    if (vbase + total > a.nnz) {  // only reachable through an inconsistent RankIndex
        if (tid == 0) latch_status(a.hdr, ENDOR_ERR_CORRUPTION);
        return;
    }
    const uintptr_t vlo = reinterpret_cast<uintptr_t>(a.values);
    const uintptr_t vhi = vlo + a.nnz * EB;
    const uintptr_t wstart = vlo + vbase * EB;
    const uintptr_t wend = wstart + uint64_t(total) * EB;
    const uintptr_t astart = wstart & ~uintptr_t(15);
    const uint32_t nvec = uint32_t((wend - astart + 15) >> 4);
    for (uint32_t v = tid; v < nvec; v += kExpandThreads) {
        const uintptr_t addr = astart + uintptr_t(v) * 16;
        uint4 q;
        if (addr >= vlo && addr + 16 <= vhi) {
            q = __ldg(reinterpret_cast<const uint4*>(addr));
        } else {  // first/last partial block of the whole values buffer
            uint32_t r[4] = {0u, 0u, 0u, 0u};
            for (int b = 0; b < 16; ++b) {
                const uintptr_t x = addr + b;
                if (x >= vlo && x < vhi) r[b >> 2] |= uint32_t(*reinterpret_cast<const uint8_t*>(x)) << ((b & 3) * 8);
            }
            q = make_uint4(r[0], r[1], r[2], r[3]);
        }
        *reinterpret_cast<uint4*>(s_vals + v * 16) = q;
    }
    const uint32_t off = uint32_t(wstart - astart);
    __syncthreads();

    // expand: chunk c covers elements [c*EPC, c*EPC+EPC) of the tile
    const uint32_t nchunks = (count + EPC - 1) / EPC;
    uint8_t* out = a.dst + t0 * EB;
    const bool aligned = (EB == 1) || ((off & 1u) == 0);
    for (uint32_t c = tid; c < nchunks; c += kExpandThreads) {
        const uint32_t e = c * EPC, wi = e >> 5, sh = e & 31;
        const uint32_t word = s_word[wi];
        const uint32_t m = (word >> sh) & CMASK;
        const uint32_t r = s_wpre[wi] + __popc(word & ((1u << sh) - 1u));
        const uint32_t p = off + r * EB;
        const uint4 q = aligned ? gather_chunk<EB, true>(m, p, s_vals)
                                : gather_chunk<EB, false>(m, p, s_vals);
        if (e + EPC <= count) {
            *reinterpret_cast<uint4*>(out + uint64_t(e) * EB) = q;
        } else {  // ragged tail of the range
            const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (uint32_t b = 0; b < 16; ++b)
                if (b < (count - e) * EB) out[uint64_t(e) * EB + b] = uint8_t(qw[b >> 2] >> ((b & 3) * 8));
        }
    }
}

// ---------------------------------------------------------------------------
// host-side launchers (used by capi.cpp)
// ---------------------------------------------------------------------------
cudaError_t launch_scan(const ScanArgs& in, cudaStream_t s) {
    ScanArgs a = in;
    const uint64_t words = (a.e1 + 31) / 32 - a.e0 / 32;
    a.nblocks = uint32_t(ceil_div(words, kScanBlockWords));
    if (a.nblocks == 0) return cudaSuccess;
    scan_kernel<<<a.nblocks, kScanThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_expand(const ExpandArgs& a, int eb, cudaStream_t s) {
    const uint64_t ntiles = ceil_div(a.e1 - a.e0, kTileElems);
    if (ntiles == 0) return cudaSuccess;
    if (eb == 2) expand_kernel<2><<<unsigned(ntiles), kExpandThreads, 0, s>>>(a);
    else expand_kernel<1><<<unsigned(ntiles), kExpandThreads, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace endor_b200
