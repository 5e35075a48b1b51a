// scan.cu -- rank (prefix-popcount) kernels: the GPU form of the reference's
// serial value cursor and of build_rank_index (bitmap.hpp:117-132).
//
//   count_kernel   hot path.  Two-level, no inter-CTA waiting: every CTA
//                  popcounts a contiguous range of 262144-bit count blocks
//                  (streamed through a 2-stage TMA bulk ring), writes the
//                  CTA-local exclusive offset of each 1024-bit sub-tile and
//                  its aggregate; the last CTA to finish scans the aggregates
//                  into per-CTA bases and checks the total against nnz
//                  (codec.hpp:158-160).  Reads the bitmap once (n/8 bytes).
//   scan_kernel    general form: arbitrary [e0, e1) ranges with a base
//                  offset, decoupled look-back across CTAs, writing or
//                  verifying a caller's RankIndex at its chunk size
//                  (check_index, codec.hpp:170-184) -- used by
//                  build_rank_index, decompress_chunked and
//                  decompress_chunk_into.
//
// HBM-bound integer kernels (no tensor cores: no GEMM-shaped work here).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace endor_b200 {

// ---------------------------------------------------------------------------
// count_kernel (batched)
// ---------------------------------------------------------------------------
#ifdef ENDOR_CTA_TIMING  // development aid (tools/count_timeline.py): per-CTA phase timestamps
__device__ unsigned long long g_count_times[8 * 4096];
#define CT_STAMP(k)                                                                        \
    do {                                                                                   \
        if (threadIdx.x == 0) {                                                            \
            unsigned long long t_;                                                         \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                         \
            g_count_times[8 * blockIdx.x + (k)] = t_;                                      \
        }                                                                                  \
    } while (0)
extern "C" int endor_debug_count_times(unsigned long long* host_out, int n) {
    return int(cudaMemcpyFromSymbol(host_out, g_count_times, sizeof(unsigned long long) * 8 * n));
}
#else
#define CT_STAMP(k) \
    do {            \
    } while (0)
#endif
__global__ void __launch_bounds__(kScanThreads) count_kernel(const __grid_constant__ Batch b) {
    CT_STAMP(0);
    constexpr int kVecPerThread = kCountBlockWords / 4 / kScanThreads;  // uint4 per thread per block
    static_assert(kVecPerThread * kScanThreads * 4 == kCountBlockWords, "block / thread geometry");
    __shared__ uint32_t s_sub[2][kCountSubs];  // double-buffered: one barrier per block
    __shared__ int s_last;
    __shared__ __align__(8) unsigned long long s_full[kCountStages];
    extern __shared__ __align__(128) uint4 s_blk[];  // [kCountStages][kCountBlockWords / 4]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ti = batch_tensor_of_cblk(b, blockIdx.x);
    const BatchTensor& T = b.t[ti];
    const uint32_t lc = blockIdx.x - T.cblk0;  // CTA index within the tensor
    const uint64_t n = T.n, nbytes = (n + 7) / 8;
    const uint64_t nwords = (n + 31) / 32;
    const uint64_t nblocks = ceil_div(nwords, kCountBlockWords);
    const uint64_t cb0 = uint64_t(lc) * T.cbpc, cb1 = umin64(nblocks, cb0 + T.cbpc);
    const uint64_t nsubs = (nwords + 31) / 32;
    // kCountStages-deep ring of count blocks filled by 1-D TMA bulk copies:
    // blocks cb+1 .. cb+S-1 are in flight while block cb is counted
    const uint32_t full0 = smem_u32(&s_full[0]);
    auto full_block = [&](uint64_t cb) { return cb < cb1 && (cb + 1) * kCountBlockWords * 32 <= n; };
    auto issue = [&](uint64_t cb, int st) {  // thread 0 only
        const uint32_t bar = full0 + 8 * st;
        mbar_arrive_expect_tx(bar, kCountBlockWords * 4);
        bulk_g2s(smem_u32(s_blk + st * (kCountBlockWords / 4)), T.bitmap + cb * kCountBlockWords * 4,
                 kCountBlockWords * 4, bar);
    };
    if (tid == 0) {
        for (int st = 0; st < kCountStages; ++st) mbar_init(full0 + 8 * st, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();  // every global access below may depend on the previous kernel
    CT_STAMP(1);
    pdl_launch_dependents();
    if (tid == 0)
        for (int st = 0; st < kCountStages; ++st)
            if (full_block(cb0 + st)) issue(cb0 + st, st);

    // stream this CTA's range of count blocks; sub-tile offsets are relative
    // to the range start, whose base comes from the last-CTA scan
    unsigned long long running = 0;
    int it = 0;
    for (uint64_t cb = cb0; cb < cb1; ++cb, ++it) {
        const uint64_t w0 = cb * kCountBlockWords;
        const int st = it % kCountStages;
        uint32_t* sub = s_sub[it & 1];
        if (full_block(cb)) {
            // full block: 8 consecutive lanes (128 B) = one 1024-bit sub-tile
            mbar_wait(full0 + 8 * st, (it / kCountStages) & 1);
            if (it == 0) CT_STAMP(2);
            uint4 v[kVecPerThread];
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j) v[j] = s_blk[st * (kCountBlockWords / 4) + j * kScanThreads + tid];
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j) {
                uint32_t c = __popc(v[j].x) + __popc(v[j].y) + __popc(v[j].z) + __popc(v[j].w);
                c += __shfl_xor_sync(0xffffffffu, c, 1);
                c += __shfl_xor_sync(0xffffffffu, c, 2);
                c += __shfl_xor_sync(0xffffffffu, c, 4);
                if ((lane & 7) == 0) sub[32 * j + tid / 8] = c;
            }
        } else {
            // ragged last block: word loads with the tail masked and padding checked
            for (int s = warp; s < kCountSubs; s += kScanThreads / 32) {
                const uint64_t wi = w0 + uint64_t(s) * 32 + lane;
                uint32_t wv = 0;
                if (wi < nwords) {
                    wv = load_word32(T.bitmap, wi, nbytes);
                    const uint64_t bit0 = wi * 32;
                    if (bit0 + 32 > n) {
                        const uint32_t keep = uint32_t(n - bit0);
                        if (n & 7) {  // padding bits of the final byte must be zero (bitmap.hpp:78-84)
                            const uint64_t pad_end = ((n + 7) & ~7ull) - bit0;
                            const uint32_t padmask =
                                (pad_end >= 32 ? 0xffffffffu : ((1u << pad_end) - 1u)) & ~((1u << keep) - 1u);
                            if (wv & padmask) latch_status(b.hdr, ENDOR_ERR_CORRUPTION);
                        }
                        wv &= (1u << keep) - 1u;
                    }
                }
                const uint32_t c = __reduce_add_sync(0xffffffffu, __popc(wv));
                if (lane == 0) sub[s] = c;
            }
        }
        __syncthreads();  // block cb read by every thread, sub[] complete
        // stage st is free again: refill it with the block kCountStages ahead
        if (tid == 0 && full_block(cb + kCountStages)) issue(cb + kCountStages, st);
        if (warp == 0) {  // exclusive offsets of the block's sub-tiles (kCountSubs / 32 per lane)
            constexpr int kPer = kCountSubs / 32;
            uint32_t cs[kPer], sum = 0;
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                cs[k] = sub[kPer * lane + k];
                sum += cs[k];
            }
            const uint32_t incl = warp_incl_scan(sum, lane);
            unsigned long long e = running + (incl - sum);
            const uint64_t s0 = w0 / 32 + kPer * lane;
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                if (s0 + k < nsubs) b.tsub[T.sub0 + s0 + k] = e;
                e += cs[k];
            }
            running += __shfl_sync(0xffffffffu, incl, 31);
        }
        // (no second barrier: the next block writes the other sub[] buffer, and
        // warp 0 finishes this scan before it reaches the next barrier)
    }
    CT_STAMP(3);
    if (tid == 0) {
        b.blk[T.blk0 + lc] = running;  // warp 0's lane 0 holds the range aggregate
        __threadfence();
        const unsigned long long d = atomicAdd(&b.hdr->done, 1ull);
        s_last = (d == gridDim.x - 1);
    }
    __syncthreads();
    CT_STAMP(4);
    if (!s_last) return;

    // ---- last CTA: per tensor, exclusive scan of its CTA aggregates -> bases -----
    // One warp per tensor, all tensors at once.  The aggregates are read kAggK
    // per lane at a time with independent loads (lane-strided, one L2 round
    // trip per 32 kAggK entries -- a serial per-lane loop would pay one round
    // trip per entry), scanned in registers, and rewritten as bases.
    __threadfence();
    constexpr int kAggK = 8;
    for (int i = warp; i < b.count; i += kScanThreads / 32) {
        const BatchTensor& U = b.t[i];
        if (U.idx) continue;  // caller-indexed: not counted here (expand checks its tail)
        unsigned long long* blk = b.blk + U.blk0;
        const uint32_t nb = U.ncta;  // one aggregate per count CTA of this tensor
        unsigned long long run = 0;
        for (uint32_t base = 0; base < nb; base += 32 * kAggK) {
            unsigned long long v[kAggK];
#pragma unroll
            for (int k = 0; k < kAggK; ++k) {
                const uint32_t x = base + 32 * k + lane;
                v[k] = x < nb ? __ldcg(&blk[x]) : 0ull;
            }
#pragma unroll
            for (int k = 0; k < kAggK; ++k) {
                const uint32_t x = base + 32 * k + lane;
                const unsigned long long incl = warp_incl_scan(v[k], lane);
                if (x < nb) blk[x] = run + incl - v[k];
                run += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
        if (lane == 0) {
            blk[nb] = run;  // grand total of the tensor
            b.hdr->total = run;
            if (b.check_total && run != U.nnz) latch_status(b.hdr, ENDOR_ERR_CORRUPTION);
        }
    }
    if (tid == 0) b.hdr->done = 0;
    CT_STAMP(5);
}

void batch_plan(Batch& b, uint64_t* sub_total, uint64_t* blk_total, int count_ctas) {
    uint64_t tile = 0, sub = 0, ntot = 0;
    uint32_t blk = 0, cta = 0;
    for (int i = 0; i < b.count; ++i) ntot += b.t[i].n;
    for (int i = 0; i < b.count; ++i) {
        BatchTensor& T = b.t[i];
        const uint64_t nb = ceil_div((T.n + 31) / 32, kCountBlockWords);
        // count CTAs in proportion to size (~count_ctas in total), whole blocks each
        uint64_t want = ntot ? (uint64_t(count_ctas) * T.n + ntot - 1) / ntot : 1;
        want = want < 1 ? 1 : (want > nb ? nb : want);
        T.cbpc = uint32_t(ceil_div(nb, want));
        T.ncta = T.idx ? 0u : uint32_t(ceil_div(nb, T.cbpc));  // caller-indexed: no count pass
        T.tile0 = tile;
        T.sub0 = sub;
        T.blk0 = blk;
        T.cblk0 = cta;
        tile += ceil_div(T.n, kTileElems);
        // +16: the TMA copies 8 entries per tile; keep every tensor's entries
        // 64-byte aligned (bulk-copy sources must be 16-byte aligned)
        sub += (ceil_div(T.n, kSubElems) + 16 + 7) & ~uint64_t(7);
        blk += T.ncta + 2;
        cta += T.ncta;
    }
    b.ntiles = tile;
    b.ncblk = cta;
    *sub_total = sub;
    *blk_total = blk;
}

// A caller's RankIndex at any chunk size (kDefaultChunkSize 4096,
// codec.hpp:19, or any nonzero size the RankIndex constructor accepts,
// bitmap.hpp:104) checked entry by entry: idx[k] must equal rank(k * cs)
// (bitmap.hpp:121-131), read from a 1024-element sub-tile rank table plus the
// popcount of the (< 1024) bits between the sub-tile start and k * cs.
__global__ void __launch_bounds__(256) verify_index_kernel(const unsigned long long* __restrict__ idx,
                                                           uint64_t chunks, uint64_t cs,
                                                           const uint8_t* __restrict__ bitmap, uint64_t nbytes,
                                                           const unsigned long long* __restrict__ tsub,
                                                           const unsigned long long* __restrict__ blk,
                                                           uint64_t spc, WsHeader* hdr) {
    const uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= chunks) return;
    const uint64_t p = k * cs, j = p / kSubElems;  // p < n: whole words below p exist
    unsigned long long r = tsub[j] + (blk ? blk[j / spc] : 0ull);
    uint64_t w = j * 32;
    for (; (w + 1) * 32 <= p; ++w) r += __popc(load_word32(bitmap, w, nbytes));
    if (p & 31) r += __popc(load_word32(bitmap, w, nbytes) & ((1u << (p & 31)) - 1u));
    if (idx[k] != r) latch_status(hdr, ENDOR_ERR_CORRUPTION);
}

cudaError_t launch_verify_index(const unsigned long long* idx, uint64_t chunks, uint64_t cs, const uint8_t* bitmap,
                                uint64_t n, const unsigned long long* tsub, const unsigned long long* blk,
                                uint64_t spc, WsHeader* hdr, cudaStream_t s) {
    if (chunks == 0) return cudaSuccess;
    verify_index_kernel<<<unsigned(ceil_div(chunks, 256)), 256, 0, s>>>(idx, chunks, cs, bitmap, (n + 7) / 8, tsub,
                                                                       blk, spc ? spc : 1, hdr);
    return cudaGetLastError();
}

cudaError_t launch_count(const Batch& b, cudaStream_t s) {
    if (b.ncblk == 0) return cudaSuccess;
    constexpr int smem = kCountStages * kCountBlockWords * 4;  // the TMA ring
    cudaError_t e = kernel_slots(reinterpret_cast<const void*>(count_kernel), kScanThreads, smem, nullptr, nullptr);
    if (e != cudaSuccess) return e;
    return launch_pdl(count_kernel, dim3(b.ncblk), dim3(kScanThreads), smem, s, b);
}

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
            if (bit0 < a.lo) v &= ~0u << (a.lo - bit0);  // below the range start (0 < lo - bit0 < 32)
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

    // ---- phase 2: block aggregate + warp-parallel decoupled look-back -----------
    if (warp == 0) {
        unsigned long long agg = 0;
        if (lane == 0) {
            for (int i = 0; i < kScanThreads / 32; ++i) {
                const unsigned long long t = s_warp_tot[i];
                s_warp_tot[i] = agg;  // now the warp's exclusive offset within the block
                agg += t;
            }
            lb_store(&a.lookback[blk], (blk == 0 ? kLbPrefix : kLbAgg) | (agg & kLbValue));
        }
        agg = __shfl_sync(0xffffffffu, agg, 0);
        unsigned long long excl = 0;
        if (blk > 0) {
            // window of 32 predecessors per step: lane i looks at block j - i
            for (int64_t j = int64_t(blk) - 1;;) {
                const int64_t idx = j - lane;
                const unsigned long long s = idx >= 0 ? lb_load(&a.lookback[idx]) : kLbPrefix;
                const unsigned long long f = s & ~kLbValue;
                const uint32_t pmask = __ballot_sync(0xffffffffu, f == kLbPrefix);
                const uint32_t imask = __ballot_sync(0xffffffffu, f == 0);
                const int limit = pmask ? __ffs(pmask) - 1 : 31;  // nearest inclusive prefix
                if (imask & ((2u << limit) - 1u)) continue;       // someone not published: re-poll
                unsigned long long v = lane <= limit ? (s & kLbValue) : 0ull;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
                excl += v;
                if (pmask) break;
                j -= 32;
            }
            if (lane == 0) lb_store(&a.lookback[blk], kLbPrefix | ((excl + agg) & kLbValue));
        }
        if (lane == 0) {
            const unsigned long long base = a.p0_ptr ? *a.p0_ptr : a.p0;
            s_excl = base + excl;
            if (blk == a.nblocks - 1) {
                const unsigned long long total = base + excl + agg;
                if (a.total_out) *a.total_out = total;
                if (a.tsub) a.tsub[ceil_div(wend - wbase, 32)] = total;  // window end of the last tile
                a.hdr->total = total;
                if (a.check_total && total != a.expect_total) latch_status(a.hdr, ENDOR_ERR_CORRUPTION);
            }
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
            if (a.tsub && lane == 0) a.tsub[rel / 32] = excl;  // 1024-element sub-tiles
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

cudaError_t launch_scan(const ScanArgs& in, cudaStream_t s) {
    ScanArgs a = in;
    const uint64_t words = (a.e1 + 31) / 32 - a.e0 / 32;
    a.nblocks = uint32_t(ceil_div(words, kScanBlockWords));
    if (a.nblocks == 0) return cudaSuccess;
    // The look-back state's position in the workspace depends on the tensor
    // size, so a workspace reused across sizes may hold other data there:
    // clear it (and the ticket/done counters) before every scan.
    cudaError_t e = cudaMemsetAsync(a.lookback, 0, sizeof(unsigned long long) * a.nblocks, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(&a.hdr->ticket, 0, 2 * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    scan_kernel<<<a.nblocks, kScanThreads, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace endor_b200
