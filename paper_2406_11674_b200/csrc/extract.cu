// extract.cu -- selective decompression:
//
//   extract_rows  codec.hpp:239-266  gather whole rows without materialising
//                 the matrix: out row i = dense row rows[i]
//   extract_cols  codec.hpp:271-297  gather whole columns: out[r][j] =
//                 dense[r][cols[j]]
//   check_sorted_unique  codec.hpp:224-232  index validation, reference order
//                 (per position: bound first -> BoundsError, then order ->
//                 invalid_argument; the first failing position wins)
//
// Both read ranks from count_kernel's two-level table (the GPU RankIndex at
// 1024-element granularity) plus a popcount of at most 1023 bits.  Rows whose
// starts fall on 1024-element sub-tiles (cols % 1024 == 0, every catalog
// shape) run through the persistent TMA expand (expand.cu, ROWS: tile t =
// piece t % tpr of row sel[t / tpr]); other rows here stage each 8192-element
// tile's packed values in shared memory and place them with the expand
// gather.  Columns rank 4 rows' bits per CTA in shared memory and look the
// selected values up directly (8 in flight per thread).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "gather.cuh"
#include "kernels.h"

namespace endor_b200 {

// rank(p) for a bit position p of tensor T (count_kernel output in b).
__device__ __forceinline__ unsigned long long rank_at(const RankTable& rt, uint64_t p, int lane) {
    const uint64_t sub = p / kSubElems;
    unsigned long long base;
    if (sub >= rt.nsub) {
        base = rt.blk[rt.ncta];
    } else {
        base = rt.blk[sub / (uint64_t(kCountSubs) * rt.cbpc)] + rt.tsub[sub];
    }
    // + popcount of [sub*1024, p): at most 32 words, one per lane
    const uint64_t w0 = sub * 32, wp = p / 32;
    uint32_t c = 0;
    const uint64_t w = w0 + lane;
    if (w <= wp && sub < rt.nsub) {
        uint32_t v = load_word32(rt.bitmap, w, rt.nbytes);
        if (w == wp) v &= (1u << (p & 31)) - 1u;  // bits below p only
        c = __popc(v);
    }
    return base + __reduce_add_sync(0xffffffffu, c);
}

// 32 bitmap bits starting at an arbitrary bit position p (zero past nbits).
__device__ __forceinline__ uint32_t bits_at(const uint8_t* bm, uint64_t nbytes, uint64_t p) {
    const uint64_t w = p / 32;
    const uint32_t sh = p & 31;
    const uint32_t lo = load_word32(bm, w, nbytes);
    if (!sh) return lo;
    return __funnelshift_r(lo, load_word32(bm, w + 1, nbytes), sh);
}

// ---- index validation (single CTA, positions in order) ---------------------------
__global__ void __launch_bounds__(1024) validate_indices_kernel(const unsigned long long* idx, uint64_t nsel,
                                                                uint64_t limit, WsHeader* hdr) {
    constexpr int U = 8;  // positions per thread per pass, loads in flight
    __shared__ unsigned long long s_first;
    if (threadIdx.x == 0) s_first = ~0ull;
    __syncthreads();
    for (uint64_t base = 0; base < nsel; base += 1024 * U) {
        unsigned long long cur[U], prv[U], key = ~0ull;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + threadIdx.x + 1024 * u;
            cur[u] = i < nsel ? idx[i] : 0ull;
            prv[u] = i > 0 && i < nsel ? idx[i - 1] : 0ull;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + threadIdx.x + 1024 * u;
            if (i >= nsel) continue;
            if (cur[u] >= limit) key = min(key, (unsigned long long)(i * 2));                        // BoundsError
            else if (i > 0 && cur[u] <= prv[u]) key = min(key, (unsigned long long)(i * 2 + 1));     // invalid_argument
        }
        if (key != ~0ull) atomicMin(&s_first, key);
        __syncthreads();
        if (s_first != ~0ull) break;  // uniform: everyone read the same value
        __syncthreads();
    }
    if (threadIdx.x == 0 && s_first != ~0ull)
        latch_status(hdr, (s_first & 1) ? ENDOR_ERR_INVALID_ARGUMENT : ENDOR_ERR_BOUNDS);
}

// ---- one 8192-element tile of a row: bits, ranks, staged values ----------------------
// Shared by extract_rows and the tiled extract_cols: thread tid owns the
// tile's 32-bit slice tid (bits past `count` cleared); the tile's packed
// values [rank(x0), rank(x0) + total) are staged in s_vals (aligned superset,
// ragged buffer ends byte-wise).  Returns false (after latching CORRUPTION)
// when the ranks run past nnz.
struct TileRanks {
    uint32_t wv, pc, incl, wexcl, total;
    uint32_t sb;  // shared address of the tile's first packed value
};
template <int EB>
__device__ __forceinline__ bool load_tile(const RankTable& rt, const uint8_t* values, uint64_t nnz, uint64_t x0,
                                          uint32_t count, uint8_t* s_vals, uint32_t* s_warp,
                                          unsigned long long* s_base, WsHeader* hdr, TileRanks& r) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (warp == 0) {
        const unsigned long long b = rank_at(rt, x0, lane);
        if (lane == 0) *s_base = b;
    }
    uint32_t wv = 0;
    if (uint32_t(tid) * 32 < count) {
        wv = bits_at(rt.bitmap, rt.nbytes, x0 + uint64_t(tid) * 32);
        const uint32_t rem = count - uint32_t(tid) * 32;
        if (rem < 32) wv &= (1u << rem) - 1u;
    }
    r.wv = wv;
    r.pc = __popc(wv);
    r.incl = warp_incl_scan(r.pc, lane);
    if (lane == 31) s_warp[warp] = r.incl;
    __syncthreads();
    uint32_t wexcl = 0, total = 0;
#pragma unroll
    for (int k = 0; k < kExpandThreads / 32; ++k) {
        wexcl += (k < warp) ? s_warp[k] : 0u;
        total += s_warp[k];
    }
    r.wexcl = wexcl;
    r.total = total;
    const uint64_t vbase = *s_base;
    if (vbase + total > nnz) {
        if (tid == 0) latch_status(hdr, ENDOR_ERR_CORRUPTION);
        return false;
    }
    const uintptr_t vlo = reinterpret_cast<uintptr_t>(values), vhi = vlo + nnz * EB;
    const uintptr_t ws = vlo + vbase * EB, we = ws + uint64_t(total) * EB;
    const uintptr_t as = ws & ~uintptr_t(15);
    const uint32_t nvec = uint32_t((we - as + 15) >> 4);
    for (uint32_t v = tid; v < nvec; v += kExpandThreads) {
        const uintptr_t addr = as + uintptr_t(v) * 16;
        uint4 q;
        if (addr >= vlo && addr + 16 <= vhi) {
            q = __ldg(reinterpret_cast<const uint4*>(addr));
        } else {
            uint32_t w4[4] = {0u, 0u, 0u, 0u};
            for (int b = 0; b < 16; ++b) {
                const uintptr_t x = addr + b;
                if (x >= vlo && x < vhi) w4[b >> 2] |= uint32_t(*reinterpret_cast<const uint8_t*>(x)) << ((b & 3) * 8);
            }
            q = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
        *reinterpret_cast<uint4*>(s_vals + v * 16) = q;
    }
    r.sb = smem_u32(s_vals) + uint32_t(ws - as);
    return true;
}

// packed value at shared byte address a (any alignment)
template <int EB>
__device__ __forceinline__ uint32_t lds_value(uint32_t a) {
    const uint32_t w = __funnelshift_r(lds32(a & ~3u), lds32((a & ~3u) + 4), (a & 3u) * 8);
    return EB == 2 ? (w & 0xFFFFu) : (w & 0xFFu);
}

// ---- extract_rows ------------------------------------------------------------------
// CTA = (selected row i, 8192-element tile j of that row); 256 threads, one
// 32-bit slice of the row's bits each.
template <int EB>
__global__ void __launch_bounds__(kExpandThreads) extract_rows_kernel(RankTable rt, const uint8_t* values,
                                                                      uint64_t nnz, uint64_t cols,
                                                                      const unsigned long long* sel,
                                                                      uint64_t tiles_per_row, uint8_t* out,
                                                                      WsHeader* hdr) {
    __shared__ uint32_t s_warp[kExpandThreads / 32];
    __shared__ unsigned long long s_base;
    __shared__ __align__(16) uint8_t s_vals[kTileElems * EB + 64];
    if (cta_error_latched(hdr)) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    init_luts(tid);  // published by the __syncthreads in load_tile
    const uint64_t i = blockIdx.x / tiles_per_row, j = blockIdx.x % tiles_per_row;
    const uint64_t row = sel[i];
    const uint32_t count = uint32_t(umin64(kTileElems, cols - j * kTileElems));
    TileRanks r;
    if (!load_tile<EB>(rt, values, nnz, row * cols + j * kTileElems, count, s_vals, s_warp, &s_base, hdr, r))
        return;
    __syncthreads();
    uint8_t* dst = out + (i * cols + j * kTileElems) * EB;
    if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        // the expand kernels' gather: each warp places its 1024 elements with
        // the PRMT selector tables and coalesced 16-byte stores
        const int32_t wfirst = warp * kSubElems;
        if (wfirst < int32_t(count))
            expand_subtile<EB, false>(r.wv, r.incl - r.pc, r.sb + r.wexcl * EB, dst + size_t(wfirst) * EB,
                                      min(int32_t(count) - wfirst, kSubElems), lane);
        return;
    }
    // output rows not 16-byte aligned (cols * eb % 16 != 0): scatter_range
    // semantics per element (codec.hpp:136-149), element-wise stores
    dst += uint64_t(tid) * 32 * EB;
    uint32_t rk = r.wexcl + r.incl - r.pc;
    const uint32_t nel = uint32_t(tid) * 32 < count ? min(32u, count - uint32_t(tid) * 32) : 0u;
    for (uint32_t e = 0; e < nel; ++e) {
        uint32_t v = 0;
        if ((r.wv >> e) & 1u) v = lds_value<EB>(r.sb + (rk++) * EB);
        if constexpr (EB == 2) {
            reinterpret_cast<uint16_t*>(dst)[e] = uint16_t(v);
        } else {
            dst[e] = uint8_t(v);
        }
    }
}

// ---- extract_cols ----------------------------------------------------------------
// CTA = rpc consecutive rows (their bits are one contiguous bit range, so one
// scan ranks them all): the rows' bitmap words and exclusive popcounts go to
// shared memory, then each selected column is looked up in every row.  The
// per-lookup chain (sel[k] -> rank -> packed value) is dependent, so lookups
// are batched kColBatch deep per thread to keep that many loads in flight,
// and one sel[] batch serves all rpc rows.
constexpr int kColBatch = 8;

template <int EB>
__global__ void __launch_bounds__(256) extract_cols_kernel(RankTable rt, const uint8_t* values, uint64_t nnz,
                                                           uint64_t rows, uint64_t cols,
                                                           const unsigned long long* sel, uint64_t nsel,
                                                           uint32_t rpc, uint8_t* out, WsHeader* hdr) {
    extern __shared__ uint32_t s_row[];  // [rpc * words] bits, then [rpc * words] exclusive popcounts
    __shared__ uint32_t s_warp[8];
    __shared__ unsigned long long s_base;
    if (cta_error_latched(hdr)) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t r0 = uint64_t(blockIdx.x) * rpc;
    const uint32_t nr = uint32_t(umin64(rpc, rows - r0));
    const uint32_t words = uint32_t((cols + 31) / 32), nw = nr * words;
    uint32_t* s_pre = s_row + rpc * words;
    if (warp == 0) {
        const unsigned long long b = rank_at(rt, r0 * cols, lane);
        if (lane == 0) s_base = b;
    }
    // each thread ranks a contiguous run of the (row, word) sequence
    const uint32_t per = (nw + 255) / 256, w0 = min(nw, uint32_t(tid) * per), w1 = min(nw, w0 + per);
    uint32_t sum = 0;
#pragma unroll 8
    for (uint32_t w = w0; w < w1; ++w) {
        const uint32_t r = w / words, j = w - r * words;
        uint32_t v = bits_at(rt.bitmap, rt.nbytes, (r0 + r) * cols + uint64_t(j) * 32);
        const uint64_t rem = cols - uint64_t(j) * 32;
        if (rem < 32) v &= (1u << rem) - 1u;
        s_row[w] = v;
        sum += __popc(v);
    }
    const uint32_t incl = warp_incl_scan(sum, lane);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t run = incl - sum, total = 0;
    for (int k = 0; k < 8; ++k) {
        run += k < warp ? s_warp[k] : 0u;
        total += s_warp[k];
    }
    for (uint32_t w = w0; w < w1; ++w) {
        s_pre[w] = run;
        run += __popc(s_row[w]);
    }
    const unsigned long long base = s_base;
    if (base + total > nnz) {
        if (tid == 0) latch_status(hdr, ENDOR_ERR_CORRUPTION);
        return;
    }
    __syncthreads();
    for (uint64_t k0 = tid; k0 < nsel; k0 += 256 * kColBatch) {
        uint32_t w[kColBatch], msk[kColBatch];
#pragma unroll
        for (int u = 0; u < kColBatch; ++u) {
            const uint64_t k = k0 + 256 * u;
            const unsigned long long c = k < nsel ? __ldg(sel + k) : 0ull;
            w[u] = uint32_t(c / 32);
            msk[u] = k < nsel ? (1u << (c & 31)) : 0u;
        }
        for (uint32_t r = 0; r < nr; ++r) {
            uint32_t v[kColBatch];
#pragma unroll
            for (int u = 0; u < kColBatch; ++u) {
                const uint32_t word = s_row[r * words + w[u]];
                v[u] = 0;
                if (word & msk[u]) {
                    const uint64_t rk = base + s_pre[r * words + w[u]] + __popc(word & (msk[u] - 1u));
                    if constexpr (EB == 2) {
                        // the packed values may sit at any alignment (file_io.hpp:32-36)
                        v[u] = (reinterpret_cast<uintptr_t>(values) & 1)
                                   ? uint32_t(__ldg(values + rk * 2)) | (uint32_t(__ldg(values + rk * 2 + 1)) << 8)
                                   : uint32_t(__ldg(reinterpret_cast<const uint16_t*>(values) + rk));
                    } else {
                        v[u] = uint32_t(__ldg(values + rk));
                    }
                }
            }
            uint8_t* orow = out + (r0 + r) * nsel * EB;
#pragma unroll
            for (int u = 0; u < kColBatch; ++u) {
                const uint64_t k = k0 + 256 * u;
                if (k < nsel) {
                    if constexpr (EB == 2) reinterpret_cast<uint16_t*>(orow)[k] = uint16_t(v[u]);
                    else orow[k] = uint8_t(v[u]);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
cudaError_t launch_validate_indices(const unsigned long long* idx, uint64_t nsel, uint64_t limit, WsHeader* hdr,
                                    cudaStream_t s) {
    if (nsel == 0) return cudaSuccess;
    validate_indices_kernel<<<1, 1024, 0, s>>>(idx, nsel, limit, hdr);
    return cudaGetLastError();
}

cudaError_t launch_extract_rows(const RankTable& rt, const uint8_t* values, uint64_t nnz, uint64_t cols, int eb,
                                const unsigned long long* sel, uint64_t nsel, uint8_t* out, WsHeader* hdr,
                                cudaStream_t s) {
    const uint64_t tpr = ceil_div(cols, kTileElems);
    if (nsel == 0 || tpr == 0) return cudaSuccess;
    const uint64_t grid = tpr * nsel;
    if (grid > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
    if (eb == 2) extract_rows_kernel<2><<<unsigned(grid), kExpandThreads, 0, s>>>(rt, values, nnz, cols, sel, tpr, out, hdr);
    else extract_rows_kernel<1><<<unsigned(grid), kExpandThreads, 0, s>>>(rt, values, nnz, cols, sel, tpr, out, hdr);
    return cudaGetLastError();
}

cudaError_t launch_extract_cols(const RankTable& rt, const uint8_t* values, uint64_t nnz, uint64_t rows,
                                uint64_t cols, int eb, const unsigned long long* sel, uint64_t nsel, uint8_t* out,
                                WsHeader* hdr, cudaStream_t s) {
    if (rows == 0 || nsel == 0) return cudaSuccess;
    const uint64_t words = (cols + 31) / 32;
    // rows per CTA: one sel[] batch serves them all (ENDOR_EXTRACT_COLS_RPC overrides)
    static const int env_rpc = [] {
        const char* e = getenv("ENDOR_EXTRACT_COLS_RPC");
        return e ? atoi(e) : 0;
    }();
    uint64_t rpc = env_rpc > 0 ? uint64_t(env_rpc) : 4;
    while (rpc > 1 && rpc * words * 8 > 64 * 1024) rpc /= 2;
    const size_t smem = size_t(rpc * words * 8);
    cudaError_t e = kernel_slots(eb == 2 ? reinterpret_cast<const void*>(extract_cols_kernel<2>)
                                         : reinterpret_cast<const void*>(extract_cols_kernel<1>),
                                 256, 200 * 1024, nullptr, nullptr);
    if (e != cudaSuccess) return e;
    const uint64_t grid = ceil_div(rows, rpc);
    if (grid > 0x7FFFFFFFull || smem > 200 * 1024) return cudaErrorInvalidConfiguration;
    if (eb == 2)
        extract_cols_kernel<2><<<unsigned(grid), 256, smem, s>>>(rt, values, nnz, rows, cols, sel, nsel,
                                                                 uint32_t(rpc), out, hdr);
    else
        extract_cols_kernel<1><<<unsigned(grid), 256, smem, s>>>(rt, values, nnz, rows, cols, sel, nsel,
                                                                 uint32_t(rpc), out, hdr);
    return cudaGetLastError();
}

}  // namespace endor_b200
