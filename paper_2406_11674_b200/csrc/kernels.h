// kernels.h -- launch interfaces of the sm_100a kernels (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace endor_b200 {

struct ScanArgs {
    const uint8_t* bitmap;
    uint64_t nbytes;         // ceil(n/8): readable bitmap bytes
    uint64_t n;              // tensor element count (padding check)
    uint64_t e0, e1;         // bit range [e0, e1), e0 % 64 == 0
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
    uint64_t e0, e1;
    const unsigned long long* tprefix;  // per-tile offsets (fallback kernel)
    const unsigned long long* tsub;     // CTA-local sub-tile offsets from count_kernel (TMA kernel)
    const unsigned long long* blk;      // count-CTA bases, total at [nblk] (TMA kernel)
    uint8_t* dst;  // base of the full dense matrix
    WsHeader* hdr;
};

// count_kernel: two-level popcount of a whole bitmap [0, n).
struct CountArgs {
    const uint8_t* bitmap;
    uint64_t nbytes;
    uint64_t n;
    unsigned long long* tsub;  // CTA-local exclusive offset per 1024-bit sub-tile
    unsigned long long* blk;   // per-CTA aggregates -> exclusive bases; total at [nblk]
    int check_total;
    uint64_t expect_total;
    WsHeader* hdr;
};
cudaError_t launch_count(const CountArgs& a, cudaStream_t s);

cudaError_t launch_scan(const ScanArgs& a, cudaStream_t s);
cudaError_t launch_expand(const ExpandArgs& a, int eb, cudaStream_t s);
cudaError_t launch_expand_tma(const ExpandArgs& a, int eb, cudaStream_t s);
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

}  // namespace endor_b200
