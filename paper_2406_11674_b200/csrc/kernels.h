// kernels.h -- launch interfaces of the sm_100a kernels (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "common.cuh"

namespace endor_b200 {

// thread-local last-error detail of the C ABI (capi.cu); returns code
int set_last_error(int code, const char* what);

// One-time, per-device kernel setup (cudaFuncSetAttribute is per device):
// raises the dynamic shared-memory limit of `fn` to `smem` on the current
// device and returns its resident CTAs per SM at `threads` and the SM count.
// Thread-safe; cached per (kernel, device).
cudaError_t kernel_slots(const void* fn, int threads, size_t smem, int* blocks_per_sm, int* sms);

// Launch with programmatic dependent launch (see pdl_wait in common.cuh):
// the kernel must call pdl_wait() before touching global memory that the
// previous kernel in the stream may write.  ENDOR_PDL=0 launches plainly.
bool pdl_enabled();
template <typename... Params, typename... Args>
cudaError_t launch_pdl(void (*kernel)(Params...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

struct ScanArgs {
    const uint8_t* bitmap;
    uint64_t nbytes;         // ceil(n/8): readable bitmap bytes
    uint64_t n;              // tensor element count (padding check)
    uint64_t e0, e1;         // bit range [e0, e1), e0 % 32 == 0
    uint64_t lo;             // first counted bit (e0 <= lo < e0 + 32): bits below are masked out
                             // (chunk ranges at arbitrary RankIndex chunk sizes); 0 = e0
    const unsigned long long* p0_ptr;  // base offset = *p0_ptr if set, else p0
    uint64_t p0;
    unsigned long long* tprefix;       // per-tile (relative to e0) offsets, or null
    unsigned long long* tsub;          // per-1024-element sub-tile offsets (+ total at the end), or null
    uint64_t cs;                       // chunk size for idx_out/idx_in (0 = none)
    unsigned long long* idx_out;       // write prefix at every chunk start in range
    const unsigned long long* idx_in;  // verify prefix at every chunk start in range
    int check_total;                   // verify base + count == expect_total
    uint64_t expect_total;
    unsigned long long* total_out;     // base + count (device), or null
    unsigned long long* lookback;
    WsHeader* hdr;
    uint32_t nblocks;
};

struct ExpandArgs {
    const uint8_t* bitmap;
    uint64_t nbytes;
    const uint8_t* values;
    uint64_t nnz;
    uint64_t e0, e1;                    // tiles start at e0 (e0 % 32 == 0)
    uint64_t lo;                        // first element written (e0 <= lo < e0 + 32); 0 = e0
    const unsigned long long* tprefix;  // per-tile offsets (fallback kernel)
    const unsigned long long* tsub;     // CTA-local sub-tile offsets from count_kernel (TMA kernel)
    const unsigned long long* blk;      // count-CTA bases, total at [nblk] (TMA kernel)
    uint8_t* dst;  // base of the full dense matrix
    WsHeader* hdr;
    float scale;        // dequant mode only (see BatchTensor)
    uint32_t deq_fast;
};

// ---- the hot path: a batch of whole tensors (one layer's ops) -----------------
// count_kernel + expand_tma_kernel take the batch by value (__grid_constant__),
// so one launch of each covers every tensor with no descriptor upload.
constexpr int kMaxBatch = 64;  // e.g. every row shard of 8 decoder layers (48 tensors) in one launch
struct BatchTensor {
    const uint8_t* bitmap;  // 16-byte aligned, ceil(n/8) bytes
    const uint8_t* values;  // nnz*eb bytes, any alignment
    uint8_t* dst;           // 16-byte aligned, n*eb bytes
    uint64_t n, nnz;
    uint64_t tile0;         // first global expand tile of this tensor
    uint64_t sub0;          // offset of its sub-tile entries in Batch::tsub
    uint32_t blk0;          // offset of its count-CTA entries in Batch::blk (ncta + 1 used)
    uint32_t cblk0;         // first global count CTA of this tensor
    uint32_t cbpc;          // 262144-bit count blocks per count CTA (a contiguous range)
    uint32_t ncta;          // count CTAs of this tensor
    // decompress_chunked fast path: a caller's RankIndex at chunk size 1024
    // (absolute offsets, idx[k] = rank(1024 k)); when set, no count pass runs
    // and tsub/blk are unused for this tensor.
    const unsigned long long* idx;
    uint32_t idx_subs;      // coarse-index expand (launch_expand_tma_derive): 1024-element sub-tiles per idx entry
    float scale;            // dequant mode: f16 = f32_to_f16(float(q) * scale)
    uint32_t deq_fast;      // dequant mode: scale finite with its sign bit clear
    // fused GEMV mode: y = W x with W this tensor (rows = outputs, cols % 1024 == 0);
    // each 1024-element sub-tile's dot product lands in part[sub0 + sub]
    const void* x;          // f16 [cols]
    float* part;            // fp32 partials, one per sub-tile
    uint64_t cols;
    uint64_t item0;         // fused GEMV: first work item (8 rows x 1024 cols) of this tensor
};
struct Batch {
    BatchTensor t[kMaxBatch];
    int count;
    int check_total;        // latch CORRUPTION when a popcount != nnz (codec.hpp:158-160)
    uint64_t ntiles;        // expand tiles over all tensors
    uint32_t ncblk;         // count CTAs over all tensors
    unsigned long long* tsub;  // CTA-local exclusive offset per 1024-element sub-tile
    unsigned long long* blk;   // per-count-CTA aggregates -> exclusive bases; total at [nblk]
    WsHeader* hdr;
    // extract_rows through the TMA expand (launch_expand_tma_rows): tensor 0's
    // rows sel[0..nsel) -> output rows 0..nsel; tile t = (t / tpr, t % tpr)
    const unsigned long long* sel;
    uint64_t rcols;
    uint32_t tpr;
};
__host__ __device__ inline int batch_tensor_of_tile(const Batch& b, uint64_t tile) {
    int i = b.count - 1;
    while (i > 0 && tile < b.t[i].tile0) --i;
    return i;
}
__host__ __device__ inline int batch_tensor_of_cblk(const Batch& b, uint32_t g) {
    int i = b.count - 1;
    while (i > 0 && g < b.t[i].cblk0) --i;
    return i;
}
// Fill the per-tensor offsets; returns the tsub / blk entries the batch needs
// (ws_layout_caps capacities).
void batch_plan(Batch& b, uint64_t* sub_total, uint64_t* blk_total, int count_ctas);
cudaError_t launch_count(const Batch& b, cudaStream_t s);
// check every entry of a caller's RankIndex (any chunk size cs >= 1) against
// ranks from a 1024-element sub-tile table: rank(1024 j) = (blk ? blk[j / spc]
// : 0) + tsub[j] (count_kernel's two levels, or scan_kernel's flat tsub), plus
// the popcount of the bits from the sub-tile start; latches CORRUPTION
cudaError_t launch_verify_index(const unsigned long long* idx, uint64_t chunks, uint64_t cs, const uint8_t* bitmap,
                                uint64_t n, const unsigned long long* tsub, const unsigned long long* blk,
                                uint64_t spc, WsHeader* hdr, cudaStream_t s);
cudaError_t launch_expand_tma(const Batch& b, int mode, cudaStream_t s);  // 1 i8, 2 f16, 3 dequant
cudaError_t launch_expand_tma_derive(const Batch& b, int mode, cudaStream_t s);  // idx at 2048/4096/8192
cudaError_t launch_expand_tma_rows(const Batch& b, int mode, cudaStream_t s);  // extract_rows (count tables)
// fused decompress -> GEMV over a batch (f16, cols % 1024 == 0, part set per tensor),
// then y[r] = sum of row r's cols/1024 segment partials in a fixed order
cudaError_t launch_gemv_fused(Batch& b, cudaStream_t s);
cudaError_t launch_row_reduce_batch(const Batch& b, float* const* y32, void* const* y16, cudaStream_t s);

// Rank lookups over count_kernel's two-level table for one tensor.
struct RankTable {
    const uint8_t* bitmap;
    uint64_t nbytes;
    const unsigned long long* tsub;  // CTA-range-local sub-tile offsets
    const unsigned long long* blk;   // per-count-CTA bases; blk[ncta] = total
    uint32_t cbpc, ncta;
    uint64_t nsub;
};
cudaError_t launch_validate_indices(const unsigned long long* idx, uint64_t nsel, uint64_t limit, WsHeader* hdr,
                                    cudaStream_t s);
cudaError_t launch_extract_rows(const RankTable& rt, const uint8_t* values, uint64_t nnz, uint64_t cols, int eb,
                                const unsigned long long* sel, uint64_t nsel, uint8_t* out, WsHeader* hdr,
                                cudaStream_t s);
cudaError_t launch_extract_cols(const RankTable& rt, const uint8_t* values, uint64_t nnz, uint64_t rows,
                                uint64_t cols, int eb, const unsigned long long* sel, uint64_t nsel, uint8_t* out,
                                WsHeader* hdr, cudaStream_t s);

cudaError_t launch_scan(const ScanArgs& a, cudaStream_t s);
cudaError_t launch_expand(const ExpandArgs& a, int mode, cudaStream_t s);  // mode 1 i8, 2 f16, 3 dequant
cudaError_t launch_dequant_values(const void* q, uint64_t nnz, float scale, void* out, cudaStream_t s);
cudaError_t launch_synth(uint64_t i0, uint64_t count, int eb, uint64_t seed, void* out,
                         cudaStream_t s);
cudaError_t launch_prune(uint8_t* w, uint64_t n, int eb, uint64_t target, const WsLayout& L,
                         cudaStream_t s);
cudaError_t launch_bitmap(const void* dense, uint64_t n, int eb, void* bitmap, const WsLayout& L,
                          cudaStream_t s);
cudaError_t launch_compact(const void* dense, uint64_t n, int eb, const void* bitmap,
                           const WsLayout& L, void* values, cudaStream_t s);
cudaError_t launch_gemv(uint64_t rows, uint64_t cols, const void* w, const void* x, float* y32,
                        void* y16, cudaStream_t s);
// dense GEMV over a batch: cols % 8 == 0, 16-byte aligned W and x
struct GemvBatch {
    const void* w[kMaxBatch];
    const void* x[kMaxBatch];
    float* y32[kMaxBatch];
    void* y16[kMaxBatch];
    uint64_t rows[kMaxBatch], cols[kMaxBatch];
    uint64_t warp0[kMaxBatch + 1];  // filled by launch_gemv_batch
    int count;
};
cudaError_t launch_gemv_batch(GemvBatch& gb, cudaStream_t s);
cudaError_t launch_quantize(const void* vals, uint64_t nnz, void* q, float* scale_dev, unsigned int* amax,
                            cudaStream_t s);


// ---- fused decompress -> GEMM (gemm_fused.cu, tcgen05) ------------------------
// Y[t, r] = sum_c W[r, c] X[t, c]: f16 W (Endor format) and X [tokens][x_ld],
// fp32 accumulation in TMEM; 128-row W tiles x bn tokens, K split so the grid
// fills the SMs (split partials summed in order by a second kernel).
struct GemmPlan {
    int bn;                       // UMMA N: 64, 128 or 256
    uint32_t m_tiles, n_tiles, ksplit, sps;
    uint64_t nspans;              // 128-column spans per row
    uint64_t part_bytes;          // split-K partials (0 when ksplit == 1)
    bool two_pass;                // decompress W to HBM, then the dense tcgen05 GEMM (large token counts)
};
GemmPlan gemm_plan(uint64_t rows, uint64_t cols, uint64_t tokens, int sms);
struct GemmLaunch {
    const uint8_t* bitmap;
    const uint8_t* values;
    uint64_t nnz, rows, cols, tokens;
    const unsigned long long* idx;  // flat RankIndex at chunk 1024 (absolute)
    const void* x;                  // f16 [tokens][x_ld], 16-byte aligned, x_ld * 2 % 16 == 0
    uint64_t x_ld;
    float* part;                    // plan.part_bytes of workspace
    float* y32;                     // [tokens][rows], or null
    void* y16;                      // [tokens][rows] f16, or null
    WsHeader* hdr;
    const void* w_dense;            // set: W already dense in HBM (f16 [rows][cols], cols % 8 == 0) -> dense kernel
};
cudaError_t launch_gemm_fused(const GemmPlan& p, const GemmLaunch& g, cudaStream_t s);
// count_kernel's two-level offsets -> a flat absolute 1024-chunk table, in place
// (tsub[j] += blk[j / spc] for j < count)
cudaError_t launch_flatten(unsigned long long* tsub, const unsigned long long* blk, uint64_t spc, uint64_t count,
                           cudaStream_t s);

}  // namespace endor_b200
