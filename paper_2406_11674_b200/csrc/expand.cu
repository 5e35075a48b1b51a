// expand.cu -- the Endor decompress (expand) kernels for sm_100a.
//
// detail::scatter_range (codec.hpp:132-152) writes dense[i] = bit_i ?
// values[rank(i)] : +0 one set bit at a time with a serial value cursor.  On
// the GPU the cursor becomes prefix sums (scan.cu gives every 1024-element
// sub-tile its value offset) and the per-element branch becomes a
// table-driven byte permutation:
//
//   for each 4-element nibble q of the bitmap, the up-to-4 packed values it
//   consumes are fetched as one unaligned 8-byte window (3 LDS.32 + 2 funnel
//   shifts) and PRMT places them into their slots, zeros elsewhere, using a
//   16-entry selector table (kLut) -- ~3 instructions per output element,
//   branch-free, for any byte alignment of the values stream.
//
// expand_tma_kernel (the hot path): persistent, warp-specialised.  One
// producer warp streams each 8192-element tile's bitmap (1 KiB) and its
// packed-values window into a 5-stage shared-memory ring with 1-D TMA bulk
// copies (cp.async.bulk + mbarrier complete_tx), and stages the tile's eight
// sub-tile starts (validated, relative to the window); eight consumer warps
// each expand one 1024-element sub-tile per tile, fully independently and
// with no checks on their critical path, and write dense rows with coalesced
// 16-byte stores.  HBM traffic per element: 1/8 (bitmap) + (1-s)*eb (values)
// read, eb written.
//
// expand_kernel (fallback): one CTA per tile, plain loads; used for
// decompress_chunk_into's partial ranges (which may start and end inside a
// bitmap word at arbitrary chunk sizes) and bitmaps that are not 16-byte
// aligned.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "gather.cuh"
#include "kernels.h"

namespace endor_b200 {

// ---------------------------------------------------------------------------
// persistent TMA kernel (batched over whole tensors)
// ---------------------------------------------------------------------------
// One CTA per SM holding kPipes independent pipelines (a producer warp + 8
// consumer warps + a kStages-deep ring each).  The SM's tiles -- tile
// blockIdx.x + j * gridDim.x for j = 0, 1, .. -- are claimed one at a time
// from a shared-memory counter by whichever producer is ready, so the two
// pipelines finish within a few tiles of each other.  (Two independent CTAs
// per SM with a fixed half of the tiles each did not: the warp scheduler
// favours the older CTA, which finished at 0.75x of the kernel time while
// its neighbour ran alone for the rest, tools/cta_timing.py.)
#ifndef ENDOR_TMA_PIPES
#define ENDOR_TMA_PIPES 2
#endif
#ifndef ENDOR_TMA_STAGES
#define ENDOR_TMA_STAGES 5  // per pipe: 5 x 17.6 KB (f16); 4 / 5 / 6 / 7 measured 3590 / 3950 / 3904 / 3115 dense-GB/s in r1
#endif
#ifndef ENDOR_TMA_BATCH
#define ENDOR_TMA_BATCH 6  // tiles per claim: 2 / 4 / 5 / 6 / 7 / 8 / 10 / 12 measured, 6 best (profiles/r02/claim_size_sweep.txt)
#endif
#ifndef ENDOR_TMA_LOOKAHEAD
#define ENDOR_TMA_LOOKAHEAD 2  // claims in flight per producer: their index loads land meanwhile
#endif
// Tile claims: each SM first works through its own static sequence
// (blockIdx.x + j * grid, claimed from a shared-memory counter: no global
// round trip at the start), then -- for the last ~15 % of the tiles --
// both pipes claim runs of consecutive tiles from one global pool counter.
// With a fixed 1/148 of the tiles per SM the SMs' finish times spread by ~5 %
// of a layer (tools/cta_timing.py) and the kernel ends with the slowest; an
// all-global counter balances the end but puts a round trip in front of
// every claim, which costs small tensors (profiles/r02/claim_size_sweep.txt).
// 0 = static only, for comparison.
#ifndef ENDOR_TMA_GLOBAL_CLAIMS
#define ENDOR_TMA_GLOBAL_CLAIMS 1
#endif
#ifndef ENDOR_TMA_POOL_MIN
#define ENDOR_TMA_POOL_MIN 128
#endif
#ifndef ENDOR_TMA_POOL_PCT
#define ENDOR_TMA_POOL_PCT 15
#endif
constexpr int kPipes = ENDOR_TMA_PIPES;
constexpr int kStages = ENDOR_TMA_STAGES;
constexpr int kLook = ENDOR_TMA_LOOKAHEAD;
constexpr int kBatch = ENDOR_TMA_BATCH;
constexpr int kTmaThreads = kPipes * (kConsumerWarps + 1) * 32;  // warps [0, kPipes) are the producers

template <int EB>
struct Stage {
    static constexpr uint32_t kBm = 0;                            // 1 KiB bitmap
    static constexpr uint32_t kSub = kTileElems / 8;              // 8 x u64 sub-tile offsets + abs base
    static constexpr uint32_t kVals = kSub + 128;                 // packed-values window
    static constexpr uint32_t kBytes = kVals + kTileElems * EB + 64;
};

// A caller's RankIndex is validated by the producer (monotone, within
// [0, nnz], <= 1024 values per sub-tile), so sub-tile k starts at most 1024 k
// values into the tile's window and no consumer read can leave the stage's
// 8192-value window buffer.  A middle entry that passes but disagrees with the
// bitmap yields garbage -- the reference's check_index does not look at middle
// entries either (codec.hpp:170-184) -- never an out-of-bounds access.
// header: [0, 256) mbarriers + claim counter; then per pipe kLook claims x
// kBatch tile slots of 12 u64 (a claimed tile's index entries, via cp.async)
constexpr uint32_t kSlotBytes = 16 * 8;  // 12 u64 of index entries / bases; ROWS: + the tile's sub-tile span
constexpr uint32_t kTmaHeader = 256 + ((kPipes * kLook * kBatch * kSlotBytes + 127) & ~127u);
// Coarse-index (DERIVE) kernels add, per pipe, after every pipe's stages: a
// ring of kDesc tile descriptors {tile, window start, 9 sub-tile starts}
// with its full/empty mbarriers, and the prefetched bitmaps of the claims in
// flight (kLook x kBatch x 1 KiB).
constexpr uint32_t kDesc = 8;
constexpr uint32_t kDescBytes = 64;
constexpr uint32_t kBmSlotBytes = kTileElems / 8;
constexpr uint32_t kDerivePipeBytes = 16 * kDesc + kDesc * kDescBytes + kLook * kBatch * kBmSlotBytes;
template <int EB, bool DERIVE = false>
constexpr uint32_t tma_smem_bytes() {
    return kTmaHeader + kPipes * kStages * Stage<EB>::kBytes + (DERIVE ? kPipes * kDerivePipeBytes : 0);
}
template <bool DERIVE>
constexpr int tma_threads() { return kTmaThreads + (DERIVE ? 32 * kPipes : 0); }  // + a deriver warp per pipe
static_assert(2 * kPipes * kStages * 8 + 8 <= 256, "mbarrier area");
static_assert(256 + kPipes * kLook * kSlotBytes <= kTmaHeader, "claim slot area");

#ifdef ENDOR_CTA_TIMING  // development aid (tools/cta_timing.py): per-CTA start / end globaltimer
__device__ unsigned long long g_cta_times[3 * 4096];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// DERIVE: the caller's RankIndex has a coarser chunk (2048 / 4096 / 8192 --
// the reference's default is 4096, codec.hpp:19).  A deriver warp per pipe
// takes over the claims: with each claim it also prefetches the claimed
// tiles' bitmaps (cp.async), popcounts every 1024-element sub-tile (one lane
// per sub-tile of the claim), derives the sub-tile starts from the chunk
// entries with a segmented scan, checks every entry against the bitmap
// (check_index, codec.hpp:170-184, and the middle entries, as the
// multi-launch path does), and posts one descriptor per tile to a ring; the
// pipe's TMA warp only turns descriptors into bulk copies, so a stage never
// waits behind that work, and the consumers run unchanged.
//
// ROWS: extract_rows (codec.hpp:239-266) through the same pipeline: tile t is
// 8192-element piece t % tpr of selected row sel[t / tpr] (rows start on
// 1024-element sub-tile boundaries: cols % 1024 == 0), its starts come from
// the count tables, and it lands in output row t / tpr.
template <int MODE, bool DERIVE = false, bool ROWS = false, bool POOL = false>
__global__ void __launch_bounds__(tma_threads<DERIVE>(), 1) expand_tma_kernel(const __grid_constant__ Batch b) {
    static_assert(!(DERIVE && ROWS), "row extraction reads the count tables");
#ifdef ENDOR_CTA_TIMING
    if (threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_cta_times[3 * blockIdx.x] = gtimer();
        g_cta_times[3 * blockIdx.x + 2] = smid;
    }
#endif
    constexpr int EB = mode_in(MODE), OB = mode_out(MODE);  // packed-value / dense-element bytes
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sbase = smem_u32(smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // pipe p: producer warp p, consumer warps kPipes + 8 p .. +7 (DERIVE: deriver warp kPipes * 9 + p)
    constexpr int kFirstDeriver = kPipes * (kConsumerWarps + 1);
    const bool deriver = DERIVE && warp >= kFirstDeriver;
    const int pipe = warp < kPipes ? warp : (deriver ? warp - kFirstDeriver : (warp - kPipes) / kConsumerWarps);
    const uint32_t full0 = sbase + 16 * kStages * pipe, empty0 = full0 + 8 * kStages;
    const uint32_t claim = sbase + 16 * kStages * kPipes;  // shared u32 tile-claim counter
    const uint32_t st0 = sbase + kTmaHeader + pipe * kStages * Stage<EB>::kBytes;
    const uint32_t slot0 = sbase + 256 + pipe * kLook * kBatch * kSlotBytes;  // this pipe's claim slots
    // DERIVE: this pipe's descriptor ring (full / empty barriers, descriptors) and claim bitmaps
    const uint32_t dsc0 = sbase + kTmaHeader + kPipes * kStages * Stage<EB>::kBytes + pipe * kDerivePipeBytes;
    const uint32_t dfull0 = dsc0, dempty0 = dsc0 + 8 * kDesc, desc0 = dsc0 + 16 * kDesc;
    const uint32_t bslot0 = desc0 + kDesc * kDescBytes;
    const uint64_t ntiles = b.ntiles;
    // this CTA's tiles: blockIdx.x + j * gridDim.x, j < nj
    // static claims j < jstat (a multiple of kBatch, so no claim straddles the
    // split), then pool claims: j = jstat + p, tile = grid * jstat + p
    // (POOL is chosen by the launcher: small launches -- under ENDOR_TMA_POOL_MIN
    // tiles per SM -- stay fully static, where the pool's round trips would
    // cost more than the imbalance they remove; a template parameter, so the
    // static instantiation carries none of the pool's code)
    constexpr bool pool = POOL;
    const uint32_t jstat =
        pool ? uint32_t((ntiles / gridDim.x) * (100 - ENDOR_TMA_POOL_PCT) / 100 / kBatch * kBatch) : 0u;
    const uint32_t nj = pool ? uint32_t(jstat + (ntiles - uint64_t(jstat) * gridDim.x))
                             : (blockIdx.x < ntiles ? uint32_t((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0u);

    init_luts(tid);
    if (tid == 0) {
        for (int s = 0; s < kPipes * kStages; ++s) {
            mbar_init(sbase + 16 * kStages * (s / kStages) + 8 * (s % kStages), 2);  // expect_tx + fix-up
            mbar_init(sbase + 16 * kStages * (s / kStages) + 8 * kStages + 8 * (s % kStages), kConsumerWarps);
        }
        if (DERIVE) {
            for (int p = 0; p < kPipes; ++p) {
                const uint32_t d0 = sbase + kTmaHeader + kPipes * kStages * Stage<EB>::kBytes + p * kDerivePipeBytes;
                for (uint32_t k = 0; k < kDesc; ++k) {
                    mbar_init(d0 + 8 * k, 1);               // descriptor posted
                    mbar_init(d0 + 8 * kDesc + 8 * k, 1);   // descriptor consumed
                }
            }
        }
        asm volatile("st.shared.u32 [%0], 0;" ::"r"(claim) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_wait();  // the prologue above overlapped the previous kernel's tail
    // a latched error: write nothing (the barrier inside also publishes the
    // LUTs, the claim counter and the mbarrier initialisation)
    if (cta_error_latched(b.hdr)) return;
    pdl_launch_dependents();

    if (warp < kPipes || deriver) {
        // ====== producer warp of pipe `pipe` (DERIVE: its TMA warp or its deriver warp) ======
        constexpr uint32_t kSubsPerBlk = kCountSubs;  // sub-tiles per count block
        // (tensor k's tail test runs on CTA grid - 1 - k: one test per CTA, not
        // all of a batch's on CTA 0 -- seven serial tests held CTA 0 ~4 us past
        // the others on a Llama2-70B G = 8 shard, profiles/r02/small_shard_timeline.txt)
        if (DERIVE && deriver && pipe == 0) {
            // check_index's tail test: the last chunk spans up to idx_subs sub-tiles
            for (int k = int(gridDim.x - 1 - blockIdx.x); k < b.count; k += int(gridDim.x)) {
                const BatchTensor& T = b.t[k];
                const uint64_t cs = uint64_t(T.idx_subs) * kSubElems, last = ceil_div(T.n, cs) - 1;
                const uint64_t nw = (T.n + 31) / 32, nbytes = (T.n + 7) / 8;
                uint32_t tail = 0;
                for (uint64_t w = last * cs / 32 + lane; w < nw; w += 32) {
                    uint32_t v = load_word32(T.bitmap, w, nbytes);
                    if (w * 32 + 32 > T.n) {
                        const uint32_t keep = uint32_t(T.n - w * 32);
                        if ((T.n & 7) && (v >> keep)) latch_status(b.hdr, ENDOR_ERR_CORRUPTION);
                        v &= (1u << keep) - 1u;
                    }
                    tail += __popc(v);
                }
                tail = __reduce_add_sync(0xffffffffu, tail);
                if (lane == 0 && T.idx[last] + tail != T.nnz) latch_status(b.hdr, ENDOR_ERR_CORRUPTION);
            }
        }
        // check_index's tail test (codec.hpp:177-183) for caller-indexed tensors:
        // idx[last] + popcount(last chunk) == nnz, plus the padding bits
        if (!DERIVE && pipe == 0) {
            for (int k = int(gridDim.x - 1 - blockIdx.x); k < b.count; k += int(gridDim.x)) {
                const BatchTensor& T = b.t[k];
                if (!T.idx) continue;
                const uint64_t last = ceil_div(T.n, kSubElems) - 1, w0 = last * 32;
                const uint64_t nw = (T.n + 31) / 32, nbytes = (T.n + 7) / 8;
                uint32_t v = 0;
                if (w0 + lane < nw) {
                    v = load_word32(T.bitmap, w0 + lane, nbytes);
                    const uint64_t bit0 = (w0 + lane) * 32;
                    if (bit0 + 32 > T.n) {
                        const uint32_t keep = uint32_t(T.n - bit0);
                        if ((T.n & 7) && (v >> keep)) latch_status(b.hdr, ENDOR_ERR_CORRUPTION);
                        v &= (1u << keep) - 1u;
                    }
                }
                const uint32_t tail = __reduce_add_sync(0xffffffffu, __popc(v));
                if (lane == 0 && T.idx[last] + tail != T.nnz) latch_status(b.hdr, ENDOR_ERR_CORRUPTION);
            }
        }
        // Tile t's absolute value window [s0, s1) and its nine sub-tile starts
        // relative to s0 (rel[8] = s1 - s0): the caller's RankIndex -- validated
        // here, so the consumers need no checks -- or count_kernel's two levels
        // (a tile never straddles two count CTAs' ranges).
        //
        // Tiles are claimed kBatch at a time (SM-local indices j, tile =
        // blockIdx.x + j * gridDim.x) from the shared counter; lane k < kBatch
        // fetches tile k's index entries with cp.async (global -> shared, no
        // registers: register scoreboards are per warp, so loads into one
        // register for successive claims would serialise on each other) into
        // its slot of the claim, one commit group per claim, and the claim is
        // issued kLook claims later after cp.async.wait_group(kLook - 1).
        auto tile_of = [&](uint32_t j) -> uint64_t {
            if (j >= nj) return ntiles;
            if (pool && j >= jstat) return uint64_t(jstat) * gridDim.x + (j - jstat);  // the shared pool
            return blockIdx.x + uint64_t(j) * gridDim.x;
        };
        auto fetch = [&](uint32_t slot, uint64_t t) {  // one lane per tile; t < ntiles
            const BatchTensor& T = b.t[batch_tensor_of_tile(b, t)];
            const uint64_t lt = t - T.tile0, nsub = ceil_div(T.n, kSubElems), a = lt * 8;
            auto cp8 = [&](int k, const unsigned long long* src) {
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(slot + 8 * k), "l"(src) : "memory");
            };
            if (ROWS) {  // the selected row's piece: sub-tiles [a, a + m) of tensor 0
                const uint64_t row = b.sel[t / b.tpr], j = t % b.tpr;
                const uint64_t a2 = (row * b.rcols + j * kTileElems) / kSubElems;
                const uint32_t m = uint32_t(umin64(kTileElems, b.rcols - j * kTileElems) / kSubElems);
                const uint64_t spc = uint64_t(kSubsPerBlk) * T.cbpc;  // one count CTA's range
#pragma unroll
                for (int k = 0; k <= 8; ++k)
                    if (uint32_t(k) <= m && a2 + k < nsub) cp8(k, b.tsub + T.sub0 + a2 + k);
                // range bases of entry 0 and of the piece's last sub-tile (a piece spans at most
                // two count ranges), then the base of entry m -- or the total at the tensor's end
                cp8(9, b.blk + T.blk0 + a2 / spc);
                cp8(10, b.blk + T.blk0 + (a2 + m - 1) / spc);
                cp8(11, b.blk + T.blk0 + (a2 + m < nsub ? (a2 + m) / spc : uint64_t(T.ncta)));
                asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(slot + 96), "l"(a2), "l"(uint64_t(m)) : "memory");
            } else if (DERIVE) {  // the chunk entries covering the tile and the next one's first
                const uint32_t S = T.idx_subs;
                const uint64_t nch = ceil_div(nsub, S), c0 = a / S;
#pragma unroll
                for (int k = 0; k <= 4; ++k)
                    if (uint32_t(k) * S <= 8 && c0 + k < nch) cp8(k, T.idx + c0 + k);
            } else if (T.idx) {
#pragma unroll
                for (int k = 0; k <= 8; ++k)
                    if (a + k < nsub) cp8(k, T.idx + a + k);
            } else {
                const uint64_t spc = uint64_t(kSubsPerBlk) * T.cbpc;  // one count CTA's range
#pragma unroll
                for (int k = 0; k <= 8; ++k)
                    if (a + k < nsub) cp8(k, b.tsub + T.sub0 + a + k);
                cp8(9, b.blk + T.blk0 + a / spc);                           // base of entries 0..7
                if (a + 8 < nsub) cp8(10, b.blk + T.blk0 + (a + 8) / spc);  // base of entry 8
                cp8(11, b.blk + T.blk0 + T.ncta);                           // total
            }
        };
        uint64_t src_lane = 0;  // ROWS: finish() leaves the piece's first element (of tensor 0) here
        auto finish = [&](uint32_t slot, uint64_t t, unsigned long long& s0, uint32_t* rel) {  // one lane per tile
            const BatchTensor& T = b.t[batch_tensor_of_tile(b, t)];
            const uint64_t lt = t - T.tile0, nsub = ceil_div(T.n, kSubElems), a = lt * 8;
            unsigned long long e[9];
            if (ROWS) {  // at most two count ranges per piece (8 sub-tiles < one range)
                const uint64_t a2 = lds64(slot + 96), m = lds64(slot + 104);
                src_lane = a2 * kSubElems;
                const uint64_t spc = uint64_t(kSubsPerBlk) * T.cbpc;
                const unsigned long long b0 = lds64(slot + 72), b1 = lds64(slot + 80), bm = lds64(slot + 88);
                e[0] = b0 + lds64(slot);
#pragma unroll
                for (int k = 1; k <= 8; ++k) {
                    if (uint64_t(k) < m) e[k] = ((a2 + k) / spc == a2 / spc ? b0 : b1) + lds64(slot + 8 * k);
                    else if (uint64_t(k) == m) e[k] = a2 + m < nsub ? bm + lds64(slot + 8 * k) : bm;
                    else e[k] = e[k - 1];  // past the piece: the window end
                }
                s0 = e[0];
#pragma unroll
                for (int k = 0; k <= 8; ++k) rel[k] = uint32_t(e[k] - e[0]);
                return;
            }
            if (DERIVE) {
                // chunk entries: monotone, within [0, nnz], at most one chunk of
                // values apart (clamp + latch).  rel[0..4] = the chunk starts
                // relative to the window (the window end past the tile's last
                // chunk), rel[8] = the window end; derive() fills in rel[0..7].
                const uint32_t S = T.idx_subs, m = 8 / S;
                const uint64_t nch = ceil_div(nsub, S), c0 = a / S;
                bool bad = false;
                unsigned long long lo = 0, ce[5];
#pragma unroll
                for (int k = 0; k <= 4; ++k) {
                    if (uint32_t(k) > m) {
                        ce[k] = lo;
                        continue;
                    }
                    const unsigned long long r = c0 + k < nch ? lds64(slot + 8 * k) : T.nnz;
                    unsigned long long v = r < lo ? lo : (r > T.nnz ? T.nnz : r);
                    if (k > 0 && v - lo > uint64_t(S) * kSubElems) v = lo + uint64_t(S) * kSubElems;
                    bad |= v != r;
                    ce[k] = lo = v;
                }
                if (bad) latch_status(b.hdr, ENDOR_ERR_CORRUPTION);
                s0 = ce[0];
#pragma unroll
                for (int k = 0; k <= 4; ++k) rel[k] = uint32_t(ce[k] - ce[0]);
                rel[8] = rel[4];
                return;
            }
            if (T.idx) {
                // monotone, within [0, nnz], at most 1024 values per sub-tile: clamp
                // and latch (memory safety; an entry that passes but disagrees with
                // the bitmap yields garbage like the reference)
                bool bad = false;
                unsigned long long lo = 0;
#pragma unroll
                for (int k = 0; k <= 8; ++k) {
                    const unsigned long long r = a + k < nsub ? lds64(slot + 8 * k) : T.nnz;
                    unsigned long long v = r < lo ? lo : (r > T.nnz ? T.nnz : r);
                    if (k > 0 && v - lo > kSubElems) v = lo + kSubElems;
                    bad |= v != r;
                    e[k] = lo = v;
                }
                if (bad) latch_status(b.hdr, ENDOR_ERR_CORRUPTION);
            } else {
                const unsigned long long b0 = lds64(slot + 72), tot = lds64(slot + 88);
#pragma unroll
                for (int k = 0; k < 8; ++k) e[k] = a + k < nsub ? b0 + lds64(slot + 8 * k) : tot;
                e[8] = a + 8 < nsub ? lds64(slot + 80) + lds64(slot + 64) : tot;
            }
            s0 = e[0];
#pragma unroll
            for (int k = 0; k <= 8; ++k) rel[k] = uint32_t(e[k] - e[0]);
        };
        auto claim_batch = [&](uint32_t c) -> uint32_t {  // claim c's first j (lane-uniform), fetch its tiles
            uint32_t j = 0;
            if (lane == 0) {
                asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(j) : "r"(claim), "n"(kBatch) : "memory");
                if (pool && j >= jstat)  // this SM's static run is used up: the pool
                    j = jstat + uint32_t(atomicAdd(&b.hdr->tile_claim, (unsigned long long)kBatch));
            }
            j = __shfl_sync(0xffffffffu, j, 0);
            const uint64_t t = tile_of(j + lane);
            if (lane < kBatch && t < ntiles) fetch(slot0 + ((c % kLook) * kBatch + lane) * kSlotBytes, t);
            if (DERIVE) {  // the claimed full tiles' bitmaps, 32 bytes per lane each
#pragma unroll
                for (int k = 0; k < kBatch; ++k) {
                    const uint64_t tk = tile_of(j + k);
                    if (tk >= ntiles) break;
                    const BatchTensor& T = b.t[batch_tensor_of_tile(b, tk)];
                    const uint64_t lt = tk - T.tile0;
                    if ((lt + 1) * kTileElems > T.n) continue;  // a partial tile: derive() reads global memory
                    const uint32_t dst = bslot0 + ((c % kLook) * kBatch + k) * kBmSlotBytes + 32 * lane;
                    const uint8_t* src = T.bitmap + lt * kBmSlotBytes + 32 * lane;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16), "l"(src + 16) : "memory");
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            return j;
        };
        // DERIVE: lane l takes sub-tile l % 8 of the claim's tile l / 8:
        // popcount, a segmented scan over the chunk's lanes turns the chunk
        // start into the sub-tile start, the chunk's last lane checks that the
        // chunk ends where the next entry says, and lane k gathers tile k's
        // eight starts
        static_assert(kBatch <= 32, "lane k holds claim tile k");
        // every claimer (producer warp, or the deriver with DERIVE) reports once it has
        // drawn a claim past the end; the last one resets the counter for the next launch
        auto claims_done = [&]() {
            if (pool && lane == 0) {
                const unsigned long long n_cl = uint64_t(kPipes) * gridDim.x;
                if (atomicAdd(&b.hdr->tile_done, 1ull) == n_cl - 1) {
                    b.hdr->tile_claim = 0;
                    b.hdr->tile_done = 0;
                }
            }
        };
        auto derive = [&](uint32_t c, uint32_t j0, uint32_t (&rel)[9]) {
#pragma unroll
            for (int g0 = 0; g0 < kBatch; g0 += 4) {  // four tiles (32 sub-tiles) per pass
                const int k = g0 + (lane >> 3), q = lane & 7;
                const uint64_t tk = k < kBatch ? tile_of(j0 + k) : ntiles;
                uint32_t p = 0, S = 1;
                if (tk < ntiles) {
                    const BatchTensor& T = b.t[batch_tensor_of_tile(b, tk)];
                    const uint64_t lt = tk - T.tile0;
                    const uint32_t count = uint32_t(umin64(kTileElems, T.n - lt * kTileElems));
                    S = T.idx_subs;
                    if (count == kTileElems) {
                        const uint32_t src = bslot0 + ((c % kLook) * kBatch + k) * kBmSlotBytes + 128 * q;
#pragma unroll
                        for (int v = 0; v < 8; ++v) {
                            uint32_t x0, x1, x2, x3;
                            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                         : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "r"(src + 16 * v));
                            p += __popc(x0) + __popc(x1) + __popc(x2) + __popc(x3);
                        }
                    } else {  // a partial tile (not prefetched): words from global memory, bits past the end masked
                        const uint64_t nbytes = (T.n + 7) / 8, wb = lt * (kTileElems / 32) + 32 * q;
                        for (uint32_t x = 0; x < 32; ++x) {
                            const int32_t keep = int32_t(count) - int32_t(1024 * q + 32 * x);
                            if (keep <= 0) break;
                            const uint32_t v = load_word32(T.bitmap, wb + x, nbytes);
                            p += __popc(keep >= 32 ? v : v & ((1u << keep) - 1u));
                        }
                    }
                }
                uint32_t st[5];  // tile k's chunk starts, then the window end
#pragma unroll
                for (int x = 0; x < 5; ++x) st[x] = __shfl_sync(0xffffffffu, rel[x], k < kBatch ? k : 0);
                const uint32_t cq = uint32_t(q) >> (__ffs(S) - 1), pos = uint32_t(q) & (S - 1);
                const uint32_t start = cq == 0 ? st[0] : cq == 1 ? st[1] : cq == 2 ? st[2] : st[3];
                const uint32_t next = cq == 0 ? st[1] : cq == 1 ? st[2] : cq == 2 ? st[3] : st[4];
                uint32_t x = p;
#pragma unroll
                for (uint32_t d = 1; d < 8; d <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                    if (d < S && pos >= d) x += y;
                }
                const uint32_t r = start + x - p;  // this sub-tile's first value
                if (tk < ntiles && pos == S - 1 && start + x != next) latch_status(b.hdr, ENDOR_ERR_CORRUPTION);
                const bool mine = lane >= g0 && lane < g0 + 4 && lane < kBatch;  // lane k gathers tile k's starts
                const int src0 = mine ? 8 * (lane - g0) : 0;
#pragma unroll
                for (int x2 = 0; x2 < 8; ++x2) {
                    const uint32_t v = __shfl_sync(0xffffffffu, r, src0 + x2);
                    if (mine) rel[x2] = v;
                }
            }
        };
        uint32_t qj[kLook];  // first j of the claims in flight, oldest first
        int i = 0, ti = 0;
        if (DERIVE && deriver) {
            // ---- deriver: claims, chunk entries, bitmaps, sub-tile starts -> descriptors
#pragma unroll
            for (int k = 0; k < kLook; ++k) qj[k] = claim_batch(k);
            uint32_t d = 0;
            for (uint32_t c = 0; qj[0] < nj; ++c) {
                asm volatile("cp.async.wait_group %0;" ::"n"(kLook - 1) : "memory");
                __syncwarp();
                unsigned long long tp_l = 0;
                uint32_t rel_l[9] = {};
                const uint64_t tl = tile_of(qj[0] + lane);
                if (lane < kBatch && tl < ntiles) finish(slot0 + ((c % kLook) * kBatch + lane) * kSlotBytes, tl, tp_l, rel_l);
                derive(c, qj[0], rel_l);
                __syncwarp();  // the slots are read before the claim below refills them
#pragma unroll
                for (int k = 0; k + 1 < kLook; ++k) qj[k] = qj[k + 1];
                qj[kLook - 1] = claim_batch(c + kLook);
                for (uint32_t own = 0; own < uint32_t(kBatch); ++own, ++d) {
                    const uint64_t t = __shfl_sync(0xffffffffu, tl, own);
                    if (t >= ntiles) break;
                    const uint32_t ds = d % kDesc, da = desc0 + ds * kDescBytes;
                    if (d >= kDesc) mbar_wait(dempty0 + 8 * ds, ((d / kDesc) - 1) & 1);
                    if (lane == own) {
                        asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(da), "l"(t), "l"(tp_l) : "memory");
                        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(da + 16), "r"(rel_l[0]),
                                     "r"(rel_l[1]), "r"(rel_l[2]), "r"(rel_l[3]) : "memory");
                        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(da + 32), "r"(rel_l[4]),
                                     "r"(rel_l[5]), "r"(rel_l[6]), "r"(rel_l[7]) : "memory");
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(da + 48), "r"(rel_l[8]) : "memory");
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(dfull0 + 8 * ds);
                }
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            claims_done();
            {  // end of work
                const uint32_t ds = d % kDesc, da = desc0 + ds * kDescBytes;
                if (d >= kDesc) mbar_wait(dempty0 + 8 * ds, ((d / kDesc) - 1) & 1);
                if (lane == 0) {
                    asm volatile("st.shared.u64 [%0], %1;" ::"r"(da), "l"(~0ull) : "memory");
                    mbar_arrive(dfull0 + 8 * ds);
                }
            }
            return;
        }
        if (DERIVE) {
            // ---- TMA warp: descriptors -> stages (the same stage fill as below)
            for (uint32_t d = 0;; ++d, ++i) {
                const uint32_t ds = d % kDesc, da = desc0 + ds * kDescBytes;
                mbar_wait(dfull0 + 8 * ds, (d / kDesc) & 1);
                const uint64_t t = lds64(da);
                if (t >= ntiles) break;
                const unsigned long long tp = lds64(da + 8);
                const unsigned long long te = tp + lds32(da + 48);
                uint32_t dr[8];
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(dr[0]), "=r"(dr[1]), "=r"(dr[2]),
                             "=r"(dr[3]) : "r"(da + 16));
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(dr[4]), "=r"(dr[5]), "=r"(dr[6]),
                             "=r"(dr[7]) : "r"(da + 32));
                __syncwarp();
                if (lane == 0) mbar_arrive(dempty0 + 8 * ds);  // the descriptor is in registers
            const int s = i % kStages;
            const uint32_t stg = st0 + s * Stage<EB>::kBytes;
            const uint32_t full = full0 + 8 * s;
            while (ti + 1 < b.count && t >= b.t[ti + 1].tile0) ++ti;
            const BatchTensor& T = b.t[ti];
            const uint64_t lt = t - T.tile0;
            const uintptr_t vlo = reinterpret_cast<uintptr_t>(T.values);
            const uintptr_t vhi = vlo + T.nnz * EB;
            const uintptr_t vlo16 = (vlo + 15) & ~uintptr_t(15), vhi16 = vhi & ~uintptr_t(15);
            if (i >= kStages) mbar_wait(empty0 + 8 * s, ((i / kStages) - 1) & 1);
            const uint64_t t0 = lt * kTileElems;
            const uint32_t count = uint32_t(umin64(kTileElems, T.n - t0));
            const uint32_t bm_bytes = (count + 7) / 8;
            const uint32_t bm_bulk = count == kTileElems ? 1024u : (bm_bytes & ~15u);
            const uintptr_t ws = vlo + tp * EB, we = vlo + te * EB;
            const uintptr_t as = ws & ~uintptr_t(15), ae = (we + 15) & ~uintptr_t(15);
            const uintptr_t bs = as > vlo16 ? as : vlo16, be = ae < vhi16 ? ae : vhi16;
            const uint32_t vbulk = be > bs ? uint32_t(be - bs) : 0u;
            if (lane == 0) {
                mbar_arrive_expect_tx(full, bm_bulk + vbulk);
                if (bm_bulk) bulk_g2s(stg + Stage<EB>::kBm, T.bitmap + t0 / 8, bm_bulk, full);
                if (vbulk) bulk_g2s(stg + Stage<EB>::kVals + uint32_t(bs - as), reinterpret_cast<const void*>(bs), vbulk, full);
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(stg + Stage<EB>::kSub + 64),  // window start
                             "r"(uint32_t(ws - as)) : "memory");
                asm volatile("st.shared.u64 [%0], %1;" ::"r"(stg + Stage<EB>::kSub + 72), "l"(t) : "memory");
            }
            if (lane == 0) {  // the 8 sub-tile starts, relative to the window start (from the descriptor)
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(stg + Stage<EB>::kSub), "r"(dr[0]),
                             "r"(dr[1]), "r"(dr[2]), "r"(dr[3]) : "memory");
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(stg + Stage<EB>::kSub + 16),
                             "r"(dr[4]), "r"(dr[5]), "r"(dr[6]), "r"(dr[7]) : "memory");
            }
            // edge bytes the bulk copies cannot move (the ends of the bitmap and of
            // the values buffer): only the bytes outside [bs, be) are visited
            bool edges = bm_bulk != bm_bytes;
            for (uint32_t x = bm_bulk + lane; x < bm_bytes; x += 32)
                sts8(stg + Stage<EB>::kBm + x, __ldg(T.bitmap + t0 / 8 + x));
            if (bs > ws || be < we) {
                edges = true;
                const uintptr_t h1 = vbulk ? bs : we, t1 = vbulk ? be : we;  // head [ws, h1), tail [t1, we)
                for (uintptr_t p = ws + lane; p < h1 && p < we; p += 32)
                    sts8(stg + Stage<EB>::kVals + uint32_t(p - as), *reinterpret_cast<const uint8_t*>(p));
                for (uintptr_t p = (t1 > ws ? t1 : ws) + lane; p < we; p += 32)
                    sts8(stg + Stage<EB>::kVals + uint32_t(p - as), *reinterpret_cast<const uint8_t*>(p));
            }
            if (edges) fence_proxy_async_smem();  // st.shared edges vs the TMA that later reuses the stage
            __syncwarp();
            if (lane == 0) mbar_arrive(full);
            }
        } else {
#pragma unroll
            for (int k = 0; k < kLook; ++k) qj[k] = claim_batch(k);
            for (uint32_t c = 0; qj[0] < nj; ++c) {
                asm volatile("cp.async.wait_group %0;" ::"n"(kLook - 1) : "memory");
                __syncwarp();
                unsigned long long tp_l = 0;
                uint32_t rel_l[9] = {};
                const uint64_t tl = tile_of(qj[0] + lane);
                if (lane < kBatch && tl < ntiles) finish(slot0 + ((c % kLook) * kBatch + lane) * kSlotBytes, tl, tp_l, rel_l);
                __syncwarp();  // the slots are read before the claim below refills them
#pragma unroll
                for (int k = 0; k + 1 < kLook; ++k) qj[k] = qj[k + 1];
                qj[kLook - 1] = claim_batch(c + kLook);
                for (uint32_t own = 0; own < uint32_t(kBatch); ++own, ++i) {
                const uint64_t t = __shfl_sync(0xffffffffu, tl, own);
                if (t >= ntiles) break;
                const unsigned long long tp = __shfl_sync(0xffffffffu, tp_l, own);
                const unsigned long long te = tp + __shfl_sync(0xffffffffu, rel_l[8], own);
                const int s = i % kStages;
                const uint32_t stg = st0 + s * Stage<EB>::kBytes;
                const uint32_t full = full0 + 8 * s;
                while (ti + 1 < b.count && t >= b.t[ti + 1].tile0) ++ti;
                const BatchTensor& T = b.t[ti];
                const uint64_t lt = t - T.tile0;
                const uintptr_t vlo = reinterpret_cast<uintptr_t>(T.values);
                const uintptr_t vhi = vlo + T.nnz * EB;
                const uintptr_t vlo16 = (vlo + 15) & ~uintptr_t(15), vhi16 = vhi & ~uintptr_t(15);
                const uint64_t src_t = ROWS ? __shfl_sync(0xffffffffu, src_lane, own) : 0ull;
                if (i >= kStages) mbar_wait(empty0 + 8 * s, ((i / kStages) - 1) & 1);
                const uint64_t t0 = ROWS ? src_t : lt * kTileElems;  // the tile's first element in T
                const uint32_t count = uint32_t(ROWS ? umin64(kTileElems, b.rcols - (t % b.tpr) * kTileElems)
                                                     : umin64(kTileElems, T.n - t0));
                const uint32_t bm_bytes = (count + 7) / 8;
                const uint32_t bm_bulk = count == kTileElems ? 1024u : (bm_bytes & ~15u);
                const uintptr_t ws = vlo + tp * EB, we = vlo + te * EB;
                const uintptr_t as = ws & ~uintptr_t(15), ae = (we + 15) & ~uintptr_t(15);
                const uintptr_t bs = as > vlo16 ? as : vlo16, be = ae < vhi16 ? ae : vhi16;
                const uint32_t vbulk = be > bs ? uint32_t(be - bs) : 0u;
                if (lane == 0) {
                    mbar_arrive_expect_tx(full, bm_bulk + vbulk);
                    if (bm_bulk) bulk_g2s(stg + Stage<EB>::kBm, T.bitmap + t0 / 8, bm_bulk, full);
                    if (vbulk) bulk_g2s(stg + Stage<EB>::kVals + uint32_t(bs - as), reinterpret_cast<const void*>(bs), vbulk, full);
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(stg + Stage<EB>::kSub + 64),  // window start
                                 "r"(uint32_t(ws - as)) : "memory");
                    asm volatile("st.shared.u64 [%0], %1;" ::"r"(stg + Stage<EB>::kSub + 72), "l"(t) : "memory");
                }
                if (lane == own) {  // the 8 sub-tile starts, relative to the window start
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(stg + Stage<EB>::kSub), "r"(rel_l[0]),
                                 "r"(rel_l[1]), "r"(rel_l[2]), "r"(rel_l[3]) : "memory");
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(stg + Stage<EB>::kSub + 16),
                                 "r"(rel_l[4]), "r"(rel_l[5]), "r"(rel_l[6]), "r"(rel_l[7]) : "memory");
                }
                // edge bytes the bulk copies cannot move (the ends of the bitmap and of
                // the values buffer): only the bytes outside [bs, be) are visited
                bool edges = bm_bulk != bm_bytes;
                for (uint32_t x = bm_bulk + lane; x < bm_bytes; x += 32)
                    sts8(stg + Stage<EB>::kBm + x, __ldg(T.bitmap + t0 / 8 + x));
                if (bs > ws || be < we) {
                    edges = true;
                    const uintptr_t h1 = vbulk ? bs : we, t1 = vbulk ? be : we;  // head [ws, h1), tail [t1, we)
                    for (uintptr_t p = ws + lane; p < h1 && p < we; p += 32)
                        sts8(stg + Stage<EB>::kVals + uint32_t(p - as), *reinterpret_cast<const uint8_t*>(p));
                    for (uintptr_t p = (t1 > ws ? t1 : ws) + lane; p < we; p += 32)
                        sts8(stg + Stage<EB>::kVals + uint32_t(p - as), *reinterpret_cast<const uint8_t*>(p));
                }
                if (edges) fence_proxy_async_smem();  // st.shared edges vs the TMA that later reuses the stage
                __syncwarp();
                if (lane == 0) mbar_arrive(full);
                }
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        if (!DERIVE) claims_done();  // (DERIVE: the deriver claimed)
        // end of work: a sentinel tile id releases the consumers
        {
            const int s = i % kStages;
            const uint32_t stg = st0 + s * Stage<EB>::kBytes;
            if (i >= kStages) mbar_wait(empty0 + 8 * s, ((i / kStages) - 1) & 1);
            if (lane == 0) {
                asm volatile("st.shared.u64 [%0], %1;" ::"r"(stg + Stage<EB>::kSub + 72), "l"(~0ull) : "memory");
                mbar_arrive(full0 + 8 * s);
                mbar_arrive(full0 + 8 * s);
            }
        }
    } else {
        // ================= consumer warps of pipe `pipe` =================
        const int cw = (warp - kPipes) % kConsumerWarps;
        int ti = 0;
        for (int i = 0;; ++i) {
            const int s = i % kStages;
            const uint32_t stg = st0 + s * Stage<EB>::kBytes;
            mbar_wait(full0 + 8 * s, (i / kStages) & 1);
            const uint64_t t = lds64(stg + Stage<EB>::kSub + 72);
            if (t >= ntiles) break;  // the producer's end-of-work sentinel
            while (ti + 1 < b.count && t >= b.t[ti + 1].tile0) ++ti;  // a pipe's tiles only move forward
            const BatchTensor& T = b.t[ti];
            // the tile's first element in the output: tensor T's own, or (ROWS) output row t / tpr
            const uint64_t t0 = ROWS ? (t / b.tpr) * b.rcols + (t % b.tpr) * kTileElems : (t - T.tile0) * kTileElems;
            const int32_t count = int32_t(ROWS ? umin64(kTileElems, b.rcols - (t % b.tpr) * kTileElems)
                                               : umin64(kTileElems, T.n - t0));
            const int32_t wfirst = cw * kWarpElems;
            if (wfirst < count) {
                const int32_t valid = min(count - wfirst, kWarpElems);
                const int32_t lbit = lane * 32;
                uint32_t word = 0;
                if (lane < kWarpWords && lbit < valid) {
                    word = lds32(stg + Stage<EB>::kBm + (cw * kWarpWords + lane) * 4);
                    if (valid - lbit < 32) word &= (1u << (valid - lbit)) - 1u;
                }
                const uint32_t pc = __popc(word);
                const uint32_t excl = warp_excl_scan_small(pc);
                const int sub = wfirst / kSubElems;  // this warp's 1024-element offset entry
                const uint32_t off = lds32(stg + Stage<EB>::kSub + 64);
                uint32_t rel = lds32(stg + Stage<EB>::kSub + 4 * sub);  // validated by the producer
                if (kWarpElems < kSubElems && (wfirst % kSubElems)) {
                    // second half of a 1024-element entry: skip the values of the first half
                    // (its words precede ours and are always complete)
                    uint32_t pw = 0;
                    for (int k = lane; k < (wfirst % kSubElems) / 32; k += 32)
                        pw += __popc(lds32(stg + Stage<EB>::kBm + (sub * 32 + k) * 4));
                    rel += __reduce_add_sync(0xffffffffu, pw);
                }
                const uint32_t vbase = stg + Stage<EB>::kVals + off + rel * EB;
                uint8_t* out = T.dst + (t0 + wfirst) * OB;
                if (valid == kWarpElems)
                    expand_subtile<MODE, true, kWarpElems>(word, excl, vbase, out, valid, lane, T.scale,
                                                           T.deq_fast);
                else
                    expand_subtile<MODE, false, kWarpElems>(word, excl, vbase, out, valid, lane, T.scale,
                                                            T.deq_fast);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty0 + 8 * s);
        }
    }
#ifdef ENDOR_CTA_TIMING
    __syncthreads();
    if (threadIdx.x == 0) g_cta_times[3 * blockIdx.x + 1] = gtimer();
#endif
}

// ---------------------------------------------------------------------------
// fallback: one CTA per tile, plain loads (partial ranges / unaligned bitmaps)
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kExpandThreads) expand_kernel(ExpandArgs a) {
    constexpr int EB = mode_in(MODE), OB = mode_out(MODE);  // packed-value / dense-element bytes
    __shared__ uint32_t s_warp[kExpandThreads / 32];
    __shared__ __align__(16) uint8_t s_vals[kTileElems * EB + 64];

    if (cta_error_latched(a.hdr)) return;  // a latched error: write nothing
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    init_luts(tid);
    const uint64_t t0 = a.e0 + uint64_t(blockIdx.x) * kTileElems;
    const uint64_t tend = min(a.e1, t0 + kTileElems);
    const int32_t count = int32_t(tend - t0);

    uint32_t wv = 0;
    if (tid * 32 < count) {
        wv = load_word32(a.bitmap, t0 / 32 + tid, a.nbytes);
        const int32_t rem = count - tid * 32;
        if (rem < 32) wv &= (1u << rem) - 1u;
        const uint64_t bit0 = t0 + uint64_t(tid) * 32;
        if (bit0 < a.lo) wv &= ~0u << (a.lo - bit0);  // bits before the range (scan masked them too)
    }
    const uint32_t pc = __popc(wv);
    const uint32_t incl = warp_incl_scan(pc, lane);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t wexcl = 0, total = 0;
#pragma unroll
    for (int i = 0; i < kExpandThreads / 32; ++i) {
        const uint32_t t = s_warp[i];
        wexcl += (i < warp) ? t : 0u;
        total += t;
    }

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
    __syncthreads();
    // each warp expands its own 1024 elements from the staged window
    const int32_t wfirst = warp * kSubElems;
    if (wfirst < count) {
        const uint32_t off = uint32_t(wstart - astart);
        const uint32_t vb = smem_u32(s_vals) + off + (wexcl * EB);
        const int32_t head = a.lo > t0 + wfirst ? int32_t(a.lo - (t0 + wfirst)) : 0;  // < 32
        expand_subtile<MODE, false>(wv, incl - pc, vb, a.dst + (t0 + wfirst) * OB,
                                  min(count - wfirst, kSubElems), lane, a.scale, a.deq_fast != 0, head);
    }
}

// ---------------------------------------------------------------------------
#ifdef ENDOR_CTA_TIMING
extern "C" int endor_debug_cta_times(unsigned long long* host_out, int n) {
    return int(cudaMemcpyFromSymbol(host_out, g_cta_times, sizeof(unsigned long long) * 3 * n));
}
#endif

cudaError_t launch_expand(const ExpandArgs& a, int mode, cudaStream_t s) {
    const uint64_t ntiles = ceil_div(a.e1 - a.e0, kTileElems);
    if (ntiles == 0) return cudaSuccess;
    if (mode == kModeF16) expand_kernel<kModeF16><<<unsigned(ntiles), kExpandThreads, 0, s>>>(a);
    else if (mode == kModeI8) expand_kernel<kModeI8><<<unsigned(ntiles), kExpandThreads, 0, s>>>(a);
    else expand_kernel<kModeDequant><<<unsigned(ntiles), kExpandThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int MODE, bool DERIVE = false, bool ROWS = false>
static cudaError_t launch_tma_mode(const Batch& b, cudaStream_t s) {
    constexpr uint32_t smem = tma_smem_bytes<mode_in(MODE), DERIVE>();
    constexpr int threads = tma_threads<DERIVE>();
    int blocks_per_sm = 1, sms = 148;
    cudaError_t e = kernel_slots(reinterpret_cast<const void*>(expand_tma_kernel<MODE, DERIVE, ROWS>), threads,
                                 smem, &blocks_per_sm, &sms);
    if (e != cudaSuccess) return e;
    const uint64_t grid = umin64(b.ntiles, uint64_t(blocks_per_sm) * sms);
    if (grid == 0) return cudaSuccess;
    if (ENDOR_TMA_GLOBAL_CLAIMS && b.ntiles / grid >= ENDOR_TMA_POOL_MIN) {
        // (kernel_slots also sets the pool instantiation's shared-memory limit)
        if ((e = kernel_slots(reinterpret_cast<const void*>(expand_tma_kernel<MODE, DERIVE, ROWS, true>), threads,
                              smem, nullptr, nullptr)) != cudaSuccess)
            return e;
        return launch_pdl(expand_tma_kernel<MODE, DERIVE, ROWS, true>, dim3(unsigned(grid)), dim3(threads), smem, s,
                          b);
    }
    return launch_pdl(expand_tma_kernel<MODE, DERIVE, ROWS>, dim3(unsigned(grid)), dim3(threads), smem, s, b);
}

// extract_rows (codec.hpp:239-266) through the TMA pipeline: count tables of
// tensor 0 in b.tsub / b.blk, b.sel / b.rcols / b.tpr / b.ntiles set, the
// output rows at b.t[0].dst (16-byte aligned rows: cols % 1024 == 0)
cudaError_t launch_expand_tma_rows(const Batch& b, int mode, cudaStream_t s) {
    if (mode == kModeF16) return launch_tma_mode<kModeF16, false, true>(b, s);
    return launch_tma_mode<kModeI8, false, true>(b, s);
}

// decompress_chunked with a caller's RankIndex at chunk 2048 / 4096 / 8192
// (every tensor's idx and idx_subs = chunk / 1024 set): one launch.
cudaError_t launch_expand_tma_derive(const Batch& b, int mode, cudaStream_t s) {
    if (mode == kModeF16) return launch_tma_mode<kModeF16, true>(b, s);
    return launch_tma_mode<kModeI8, true>(b, s);
}

// Whole-tensor expand of a batch through the TMA ring (needs count_kernel's
// offsets in the same workspace; 16-byte aligned bitmaps and outputs).
// mode: 1 = i8, 2 = f16 (== elem_bytes), 3 = i8 values dequantized to f16.
cudaError_t launch_expand_tma(const Batch& b, int mode, cudaStream_t s) {
    if (mode == kModeF16) return launch_tma_mode<kModeF16>(b, s);
    if (mode == kModeI8) return launch_tma_mode<kModeI8>(b, s);
    return launch_tma_mode<kModeDequant>(b, s);
}

}  // namespace endor_b200
