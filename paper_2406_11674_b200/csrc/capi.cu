// capi.cu -- the extern "C" boundary (include/endor_cuda.h): argument
// validation with the reference's error semantics, workspace layout, and
// launch sequencing.  Host code only; the kernels live in decompress.cu,
// fixtures.cu and gemv.cu.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <cstdio>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <utility>

#include "common.cuh"
#include "endor_cuda.h"
#include "kernels.h"

using namespace endor_b200;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* what) {
    g_last_error = what;
    return code;
}

}  // namespace

int endor_b200::set_last_error(int code, const char* what) {
    g_last_error = what;
    return code;
}

bool endor_b200::pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("ENDOR_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

cudaError_t endor_b200::kernel_slots(const void* fn, int threads, size_t smem, int* blocks_per_sm, int* sms) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, std::pair<int, int>> cache;  // (fn, dev) -> (bps, sms)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find({fn, dev});
    if (it == cache.end()) {
        if (smem > 48 * 1024 &&
            (e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))) != cudaSuccess)
            return e;
        int n = 0, bps = 0;
        if ((e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, threads, smem)) != cudaSuccess) return e;
        it = cache.emplace(std::make_pair(fn, dev), std::make_pair(bps < 1 ? 1 : bps, n)).first;
    }
    if (blocks_per_sm) *blocks_per_sm = it->second.first;
    if (sms) *sms = it->second.second;
    return cudaSuccess;
}

namespace {

int cuda_fail(cudaError_t e, const char* where) {
    g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
    return ENDOR_ERR_CUDA;
}

#define CK(expr)                                              \
    do {                                                      \
        cudaError_t e_ = (expr);                              \
        if (e_ != cudaSuccess) return cuda_fail(e_, #expr);   \
    } while (0)

inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// checked_element_count (dense_matrix.hpp:28-33)
inline bool checked_n(uint64_t rows, uint64_t cols, uint64_t* n) {
    if (rows != 0 && cols > UINT64_MAX / rows) return false;
    *n = rows * cols;
    return true;
}

inline int eb_of(int32_t dtype) { return dtype == ENDOR_DTYPE_F16 ? 2 : (dtype == ENDOR_DTYPE_I8 ? 1 : 0); }
inline bool is_pow2_ge64(uint64_t cs) { return cs >= 64 && (cs & (cs - 1)) == 0; }
inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

// Common validation of a tensor view; fills n / eb.
int check_view(const endor_tensor_view* t, uint64_t* n, int* eb) {
    if (!t) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null tensor view");
    *eb = eb_of(t->dtype);
    if (!*eb) return fail(ENDOR_ERR_INVALID_ARGUMENT, "unknown dtype code");
    if (!checked_n(t->rows, t->cols, n))
        return fail(ENDOR_ERR_SIZE, "matrix dimensions overflow the addressable element count");
    if (t->nnz > *n) return fail(ENDOR_ERR_CORRUPTION, "values length does not match bitmap popcount");
    if (*n > 0 && !t->bitmap) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null bitmap");
    if (t->nnz > 0 && !t->values) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null values");
    if (!aligned(t->bitmap, 4)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "bitmap must be 4-byte aligned");
    return ENDOR_OK;
}

int check_ws(void* ws, size_t ws_bytes, uint64_t n, WsLayout* L) {
    if (!ws) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null workspace");
    if (!aligned(ws, 256)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
    *L = ws_layout(ws, n);
    if (ws_bytes < L->bytes) return fail(ENDOR_ERR_INVALID_ARGUMENT, "workspace too small");
    return ENDOR_OK;
}

ScanArgs scan_args(const void* bitmap, uint64_t n, uint64_t e0, uint64_t e1, const WsLayout& L) {
    ScanArgs a{};
    a.bitmap = static_cast<const uint8_t*>(bitmap);
    a.nbytes = (n + 7) / 8;
    a.n = n;
    a.e0 = e0;
    a.e1 = e1;
    a.lookback = L.lookback;
    a.hdr = L.hdr;
    return a;
}

ExpandArgs expand_args(const endor_tensor_view* t, uint64_t n, uint64_t e0, uint64_t e1,
                       void* dst, const WsLayout& L) {
    ExpandArgs x{};
    x.bitmap = static_cast<const uint8_t*>(t->bitmap);
    x.nbytes = (n + 7) / 8;
    x.values = static_cast<const uint8_t*>(t->values);
    x.nnz = t->nnz;
    x.e0 = e0;
    x.e1 = e1;
    x.tprefix = L.tprefix;
    x.tsub = L.tsub;
    x.blk = L.blk;
    x.dst = static_cast<uint8_t*>(dst);
    x.hdr = L.hdr;
    return x;
}

// Count CTAs per batch: 3 per SM (each holds a 2 x 32 KiB TMA ring), each
// streaming a contiguous bitmap range.
// RankIndex chunk sizes the one-launch coarse-index expand takes (a tile of
// 8192 elements holds whole chunks)
bool derive_chunk(uint64_t cs) { return cs == 2048 || cs == 4096 || cs == 8192; }

int count_ctas() {
    static thread_local int dev_cached = -1, sms = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 3 * 148;
    if (dev != dev_cached) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        dev_cached = dev;
    }
    return 3 * sms;
}

// scan + expand over the whole tensor.  A 16-byte aligned bitmap takes the
// persistent TMA ring (sub-tile offsets); anything else the plain fallback.
// phase: 0 = both launches, 1 = count only, 2 = expand only (TMA path).
int full_expand(const endor_tensor_view* t, uint64_t n, int eb, void* dst, const WsLayout& L,
                ScanArgs a, cudaStream_t s, int phase = 0) {
    const ExpandArgs x = expand_args(t, n, 0, n, dst, L);
    if (aligned(t->bitmap, 16) && !a.idx_in) {
        // hot path: two-level count (no inter-CTA waits) + persistent TMA expand,
        // as a batch of one tensor
        Batch b{};
        b.count = 1;
        b.check_total = a.check_total;
        b.t[0].bitmap = static_cast<const uint8_t*>(t->bitmap);
        b.t[0].values = static_cast<const uint8_t*>(t->values);
        b.t[0].dst = static_cast<uint8_t*>(dst);
        b.t[0].n = n;
        b.t[0].nnz = t->nnz;
        uint64_t sub_cap, blk_cap;
        batch_plan(b, &sub_cap, &blk_cap, count_ctas());  // within ws_layout(n)'s capacities
        b.tsub = L.tsub;
        b.blk = L.blk;
        b.hdr = L.hdr;
        if (phase != 2) CK(launch_count(b, s));
        if (phase != 1) CK(launch_expand_tma(b, eb, s));
        return ENDOR_OK;
    }
    if (phase != 0) return fail(ENDOR_ERR_INVALID_ARGUMENT, "phase split needs a 16-byte aligned bitmap");
    // general path (verifies a caller's RankIndex / unaligned bitmap)
    a.tprefix = L.tprefix;
    CK(launch_scan(a, s));
    CK(launch_expand(x, eb, s));
    return ENDOR_OK;
}

}  // namespace

extern "C" {

int endor_cuda_abi_version(void) { return ENDOR_CUDA_ABI_VERSION; }

const char* endor_cuda_last_error_string(void) { return g_last_error.c_str(); }

const char* endor_cuda_status_name(int s) {
    switch (s) {
        case ENDOR_OK: return "OK";
        case ENDOR_ERR_SIZE: return "SizeError";
        case ENDOR_ERR_CORRUPTION: return "CorruptionError";
        case ENDOR_ERR_BOUNDS: return "BoundsError";
        case ENDOR_ERR_INVALID_ARGUMENT: return "InvalidArgument";
        case ENDOR_ERR_CUDA: return "CudaError";
        case ENDOR_ERR_CONFIG: return "ConfigError";
        case ENDOR_ERR_FORMAT: return "FormatError";
        case ENDOR_ERR_IO: return "Error";
        default: return "Unknown";
    }
}

uint64_t endor_cuda_tile_elems(void) { return kTileElems; }

size_t endor_cuda_workspace_bytes(uint64_t rows, uint64_t cols) {
    uint64_t n;
    if (!checked_n(rows, cols, &n)) return 0;
    return ws_layout(nullptr, n).bytes;
}

int endor_cuda_workspace_init(void* ws, size_t ws_bytes, void* stream) {
    if (!ws) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null workspace");
    CK(cudaMemsetAsync(ws, 0, ws_bytes, S(stream)));
    return ENDOR_OK;
}

int endor_cuda_sync_status(void* ws, void* stream) {
    if (!ws) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null workspace");
    WsHeader* hdr = static_cast<WsHeader*>(ws);
    uint32_t st = 0;
    // stream-ordered read and reset (the stream may be a non-blocking one)
    CK(cudaMemcpyAsync(&st, &hdr->status, sizeof(st), cudaMemcpyDeviceToHost, S(stream)));
    CK(cudaStreamSynchronize(S(stream)));
    if (st) {
        CK(cudaMemsetAsync(&hdr->status, 0, sizeof(uint32_t), S(stream)));
        // CTAs that saw the latched status skipped the self-resetting tile
        // pool protocol (expand.cu): start the next launch from zero
        CK(cudaMemsetAsync(&hdr->tile_claim, 0, 2 * sizeof(unsigned long long), S(stream)));
        CK(cudaStreamSynchronize(S(stream)));
        return fail(int(st), st == ENDOR_ERR_CORRUPTION
                                 ? "device check failed: bitmap popcount / rank index / padding bits "
                                   "disagree with the tensor (codec.hpp:158-160,170-184, bitmap.hpp:78-84)"
                                 : "device-latched error");
    }
    return ENDOR_OK;
}

int endor_cuda_decompress(const endor_tensor_view* t, void* dense_out, void* ws, size_t ws_bytes,
                          void* stream) {
    uint64_t n;
    int eb, st;
    if ((st = check_view(t, &n, &eb))) return st;
    if (n == 0) return ENDOR_OK;  // nnz == 0 already implied by nnz <= n
    if (!dense_out || !aligned(dense_out, 16))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "dense output must be non-null and 16-byte aligned");
    WsLayout L;
    if ((st = check_ws(ws, ws_bytes, n, &L))) return st;
    ScanArgs a = scan_args(t->bitmap, n, 0, n, L);
    a.check_total = 1;
    a.expect_total = t->nnz;
    return full_expand(t, n, eb, dense_out, L, a, S(stream));
}

static int plan_batch(const endor_tensor_view* views, void* const* outs, int count, Batch* b,
                      int* eb_out, uint64_t* nmax, size_t* bytes) {
    if (count < 0 || count > kMaxBatch || (count > 0 && !views))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "batch must hold 0..64 tensors");
    *b = Batch{};
    int eb = 0, st;
    uint64_t mx = 1;
    for (int i = 0; i < count; ++i) {
        uint64_t n;
        int e;
        if ((st = check_view(&views[i], &n, &e))) return st;
        if (eb && e != eb) return fail(ENDOR_ERR_INVALID_ARGUMENT, "batched tensors must share a dtype");
        eb = e;
        if (n && !aligned(views[i].bitmap, 16))
            return fail(ENDOR_ERR_INVALID_ARGUMENT, "batched bitmaps must be 16-byte aligned");
        if (outs && n && (!outs[i] || !aligned(outs[i], 16)))
            return fail(ENDOR_ERR_INVALID_ARGUMENT, "dense outputs must be non-null and 16-byte aligned");
        if (n == 0) continue;  // nothing to expand (nnz <= n already checked)
        BatchTensor& T = b->t[b->count++];
        T.bitmap = static_cast<const uint8_t*>(views[i].bitmap);
        T.values = static_cast<const uint8_t*>(views[i].values);
        T.dst = outs ? static_cast<uint8_t*>(outs[i]) : nullptr;
        T.n = n;
        T.nnz = views[i].nnz;
        mx = n > mx ? n : mx;
    }
    uint64_t sub_cap, blk_cap, blk_bound = 0;
    batch_plan(*b, &sub_cap, &blk_cap, count_ctas());
    for (int i = 0; i < b->count; ++i)  // size for one count CTA per block: device-independent
        blk_bound += ceil_div((b->t[i].n + 31) / 32, kCountBlockWords) + 2;
    *eb_out = eb ? eb : 2;
    *nmax = mx;
    *bytes = ws_layout_caps(nullptr, mx, sub_cap, blk_bound).bytes;
    return ENDOR_OK;
}

size_t endor_cuda_workspace_bytes_batch(const endor_tensor_view* views, int count) {
    Batch b;
    int eb;
    uint64_t nmax;
    size_t bytes = 0;
    if (plan_batch(views, nullptr, count, &b, &eb, &nmax, &bytes)) return 0;
    return bytes;
}

int endor_cuda_decompress_batch_phase(const endor_tensor_view* views, void* const* dense_outs,
                                      int count, int phase, void* ws, size_t ws_bytes, void* stream) {
    Batch b;
    if (phase < 0 || phase > 2) return fail(ENDOR_ERR_INVALID_ARGUMENT, "phase must be 0, 1 or 2");
    int eb, st;
    uint64_t nmax;
    size_t need;
    if (!dense_outs && count) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null output array");
    if ((st = plan_batch(views, dense_outs, count, &b, &eb, &nmax, &need))) return st;
    if (b.count == 0) return ENDOR_OK;
    if (!ws || !aligned(ws, 256)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
    if (ws_bytes < need) return fail(ENDOR_ERR_INVALID_ARGUMENT, "workspace too small for the batch");
    uint64_t sub_cap, blk_cap, blk_bound = 0;
    batch_plan(b, &sub_cap, &blk_cap, count_ctas());
    for (int i = 0; i < b.count; ++i) blk_bound += ceil_div((b.t[i].n + 31) / 32, kCountBlockWords) + 2;
    const WsLayout L = ws_layout_caps(ws, nmax, sub_cap, blk_bound);
    b.check_total = 1;
    b.tsub = L.tsub;
    b.blk = L.blk;
    b.hdr = L.hdr;
    if (phase != 2) CK(launch_count(b, S(stream)));
    if (phase != 1) CK(launch_expand_tma(b, eb, S(stream)));
    return ENDOR_OK;
}

int endor_cuda_decompress_batch(const endor_tensor_view* views, void* const* dense_outs, int count,
                                void* ws, size_t ws_bytes, void* stream) {
    return endor_cuda_decompress_batch_phase(views, dense_outs, count, 0, ws, ws_bytes, stream);
}

int endor_cuda_decompress_dequant(const endor_tensor_view* t, float scale, void* dense_f16_out, void* ws,
                                  size_t ws_bytes, void* stream) {
    uint64_t n;
    int eb, st;
    if ((st = check_view(t, &n, &eb))) return st;
    if (t->dtype != ENDOR_DTYPE_I8)  // codec.hpp:335-337
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "dequantize_values requires a quantized i8 tensor");
    if (n == 0) return ENDOR_OK;
    if (!dense_f16_out || !aligned(dense_f16_out, 16))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "dense output must be non-null and 16-byte aligned");
    WsLayout L;
    if ((st = check_ws(ws, ws_bytes, n, &L))) return st;
    uint32_t sbits;
    memcpy(&sbits, &scale, 4);
    // fast conversion is exact when no product can be NaN and unset slots give +0
    const uint32_t fast = ((sbits & 0x7F800000u) != 0x7F800000u) && !(sbits >> 31);
    if (aligned(t->bitmap, 16)) {
        Batch b{};
        b.count = 1;
        b.check_total = 1;
        BatchTensor& T = b.t[0];
        T.bitmap = static_cast<const uint8_t*>(t->bitmap);
        T.values = static_cast<const uint8_t*>(t->values);
        T.dst = static_cast<uint8_t*>(dense_f16_out);
        T.n = n;
        T.nnz = t->nnz;
        T.scale = scale;
        T.deq_fast = fast;
        uint64_t sub_cap, blk_cap;
        batch_plan(b, &sub_cap, &blk_cap, count_ctas());
        b.tsub = L.tsub;
        b.blk = L.blk;
        b.hdr = L.hdr;
        CK(launch_count(b, S(stream)));
        CK(launch_expand_tma(b, 3, S(stream)));
        return ENDOR_OK;
    }
    ScanArgs a = scan_args(t->bitmap, n, 0, n, L);
    a.check_total = 1;
    a.expect_total = t->nnz;
    a.tprefix = L.tprefix;
    CK(launch_scan(a, S(stream)));
    ExpandArgs x = expand_args(t, n, 0, n, dense_f16_out, L);
    x.scale = scale;
    x.deq_fast = fast;
    CK(launch_expand(x, 3, S(stream)));
    return ENDOR_OK;
}

int endor_cuda_gemv_compressed(const endor_tensor_view* t, const uint64_t* prefix1024, const void* x_f16,
                               float* y_f32, void* y_f16, void* ws, size_t ws_bytes, void* stream) {
    if (!t) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null tensor view");
    const uint64_t* pres[1] = {prefix1024};
    const void* xs[1] = {x_f16};
    float* y32[1] = {y_f32};
    void* y16[1] = {y_f16};
    if (!y_f32 && !y_f16) return fail(ENDOR_ERR_INVALID_ARGUMENT, "x must be 16-byte aligned f16[cols]; y must be given");
    return endor_cuda_gemv_compressed_batch(t, pres, xs, y32, y16, 1, ws, ws_bytes, stream);
}

int endor_cuda_gemv_compressed_batch(const endor_tensor_view* views, const uint64_t* const* prefixes1024,
                                     const void* const* x_f16, float* const* y_f32, void* const* y_f16,
                                     int count, void* ws, size_t ws_bytes, void* stream) {
    if (count < 0 || count > kMaxBatch || (count > 0 && (!views || !x_f16)))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "batch must hold 0..64 tensors with x vectors");
    for (int i = 0; i < count; ++i) {
        const endor_tensor_view* t = &views[i];
        uint64_t n;
        int eb, st;
        if ((st = check_view(t, &n, &eb))) return st;
        if (t->dtype != ENDOR_DTYPE_F16) return fail(ENDOR_ERR_INVALID_ARGUMENT, "fused GEMV needs an f16 tensor");
        if (t->cols % kSubElems)
            return fail(ENDOR_ERR_INVALID_ARGUMENT,
                        "fused GEMV needs cols % 1024 == 0 (use endor_cuda_decompress + endor_cuda_gemv)");
        if (t->rows == 0) continue;
        if (!x_f16[i] || !aligned(x_f16[i], 16) || (!(y_f32 && y_f32[i]) && !(y_f16 && y_f16[i])))
            return fail(ENDOR_ERR_INVALID_ARGUMENT, "x must be 16-byte aligned f16[cols]; y must be given");
        if (!aligned(t->bitmap, 16))
            return fail(ENDOR_ERR_INVALID_ARGUMENT, "fused GEMV needs a 16-byte aligned bitmap");
        if (prefixes1024 && prefixes1024[i] && !aligned(prefixes1024[i], 16))
            return fail(ENDOR_ERR_INVALID_ARGUMENT, "misaligned prefix");
    }
    Batch b;
    int eb, st;
    uint64_t nmax;
    size_t need;
    if ((st = plan_batch(views, nullptr, count, &b, &eb, &nmax, &need))) return st;
    if (b.count == 0) return ENDOR_OK;
    if (!ws || !aligned(ws, 256)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
    if (ws_bytes < need) return fail(ENDOR_ERR_INVALID_ARGUMENT, "workspace too small for the batch");
    // attach x / y / indices (plan_batch drops empty tensors: walk both lists)
    float* y32[kMaxBatch] = {};
    void* y16[kMaxBatch] = {};
    for (int i = 0, j = 0; i < count; ++i) {
        if (views[i].rows * views[i].cols == 0) continue;
        BatchTensor& T = b.t[j];
        T.x = x_f16[i];
        T.cols = views[i].cols;
        T.idx = prefixes1024 ? reinterpret_cast<const unsigned long long*>(prefixes1024[i]) : nullptr;
        y32[j] = y_f32 ? y_f32[i] : nullptr;
        y16[j] = y_f16 ? y_f16[i] : nullptr;
        ++j;
    }
    uint64_t sub_cap, blk_cap, blk_bound = 0;
    batch_plan(b, &sub_cap, &blk_cap, count_ctas());  // re-plan: indexed tensors need no count CTAs
    for (int i = 0; i < b.count; ++i) blk_bound += ceil_div((b.t[i].n + 31) / 32, kCountBlockWords) + 2;
    const WsLayout L = ws_layout_caps(ws, nmax, sub_cap, blk_bound);
    for (int i = 0; i < b.count; ++i) b.t[i].part = L.part + b.t[i].sub0;
    b.check_total = 1;
    b.tsub = L.tsub;
    b.blk = L.blk;
    b.hdr = L.hdr;
    CK(launch_count(b, S(stream)));  // no-op when every tensor is indexed
    CK(launch_gemv_fused(b, S(stream)));
    CK(launch_row_reduce_batch(b, y32, y16, S(stream)));
    return ENDOR_OK;
}

size_t endor_cuda_gemm_workspace_bytes(uint64_t rows, uint64_t cols, uint64_t tokens) {
    uint64_t n;
    if (!checked_n(rows, cols, &n)) return 0;
    const GemmPlan p = gemm_plan(rows, cols, tokens, count_ctas() / 3);
    return ws_layout(nullptr, n).bytes + align256(p.part_bytes) + (p.two_pass ? align256(n * 2) : 0);
}

int endor_cuda_gemm(uint64_t rows, uint64_t cols, const void* w_f16, const void* x_f16, uint64_t tokens,
                    uint64_t x_ld, float* y_f32, void* y_f16, void* ws, size_t ws_bytes, void* stream) {
    uint64_t n;
    if (!checked_n(rows, cols, &n)) return fail(ENDOR_ERR_SIZE, "matrix dimensions overflow the addressable element count");
    if (!y_f32 && !y_f16) return fail(ENDOR_ERR_INVALID_ARGUMENT, "y must be given");
    if (tokens == 0 || rows == 0) return ENDOR_OK;
    if (cols == 0) {
        if (y_f32) CK(cudaMemsetAsync(y_f32, 0, tokens * rows * 4, S(stream)));
        if (y_f16) CK(cudaMemsetAsync(y_f16, 0, tokens * rows * 2, S(stream)));
        return ENDOR_OK;
    }
    if (!w_f16 || !aligned(w_f16, 16) || cols % 8)
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "W must be a 16-byte aligned f16 [rows][cols] with cols % 8 == 0");
    if (!x_f16 || !aligned(x_f16, 16) || x_ld < cols || x_ld % 8)
        return fail(ENDOR_ERR_INVALID_ARGUMENT,
                    "x must be a 16-byte aligned f16 [tokens][x_ld] with x_ld >= cols and x_ld % 8 == 0");
    if (cols > 0x7FFFFFFFull || tokens > 0x7FFFFFFFull || rows > 0x7FFFFFFFull)
        return fail(ENDOR_ERR_SIZE, "GEMM: rows, cols and tokens must fit the TMA coordinate range (< 2^31)");
    GemmPlan p = gemm_plan(rows, cols, tokens, count_ctas() / 3);
    if (!ws || !aligned(ws, 256) || ws_bytes < 256 + align256(p.part_bytes))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "workspace too small (endor_cuda_gemm_workspace_bytes)");
    GemmLaunch g{};
    g.rows = rows;
    g.cols = cols;
    g.tokens = tokens;
    g.x = x_f16;
    g.x_ld = x_ld;
    g.part = reinterpret_cast<float*>(static_cast<char*>(ws) + 256);
    g.y32 = y_f32;
    g.y16 = y_f16;
    g.hdr = static_cast<WsHeader*>(ws);
    g.w_dense = w_f16;
    CK(launch_gemm_fused(p, g, S(stream)));
    return ENDOR_OK;
}

int endor_cuda_gemm_compressed(const endor_tensor_view* t, const uint64_t* prefix1024, const void* x_f16,
                               uint64_t tokens, uint64_t x_ld, float* y_f32, void* y_f16, void* ws, size_t ws_bytes,
                               void* stream) {
    uint64_t n;
    int eb, st;
    if ((st = check_view(t, &n, &eb))) return st;
    if (t->dtype != ENDOR_DTYPE_F16) return fail(ENDOR_ERR_INVALID_ARGUMENT, "fused GEMM needs an f16 tensor");
    if (!y_f32 && !y_f16) return fail(ENDOR_ERR_INVALID_ARGUMENT, "y must be given");
    if ((y_f32 && !aligned(y_f32, 4)) || (y_f16 && !aligned(y_f16, 2)))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "misaligned y");
    if (tokens == 0 || t->rows == 0) return ENDOR_OK;
    if (t->cols == 0) {  // empty reduction: Y = 0
        if (y_f32) CK(cudaMemsetAsync(y_f32, 0, tokens * t->rows * 4, S(stream)));
        if (y_f16) CK(cudaMemsetAsync(y_f16, 0, tokens * t->rows * 2, S(stream)));
        return ENDOR_OK;
    }
    if (!x_f16 || !aligned(x_f16, 16) || x_ld < t->cols || x_ld % 8)
        return fail(ENDOR_ERR_INVALID_ARGUMENT,
                    "x must be a 16-byte aligned f16 [tokens][x_ld] with x_ld >= cols and x_ld % 8 == 0");
    if (t->cols > 0x7FFFFFFFull || tokens > 0x7FFFFFFFull || x_ld > (uint64_t(1) << 38))
        return fail(ENDOR_ERR_SIZE, "fused GEMM: cols and tokens must fit the TMA coordinate range (< 2^31)");
    if (prefix1024 && !aligned(prefix1024, 8)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "misaligned prefix");
    WsLayout L;
    if ((st = check_ws(ws, ws_bytes, n, &L))) return st;
    const GemmPlan p = gemm_plan(t->rows, t->cols, tokens, count_ctas() / 3);
    if (ws_bytes < L.bytes + align256(p.part_bytes) + (p.two_pass ? align256(n * 2) : 0))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "workspace too small (endor_cuda_gemm_workspace_bytes)");
    const unsigned long long* idx = reinterpret_cast<const unsigned long long*>(prefix1024);
    void* wd = p.two_pass ? static_cast<char*>(ws) + L.bytes + align256(p.part_bytes) : nullptr;
    if (p.two_pass) {
        // decompress W once into the workspace (the hot path: count + TMA expand,
        // or one expand launch with the caller's index), then the dense GEMM
        Batch b{};
        b.count = 1;
        b.check_total = 1;
        b.t[0].bitmap = static_cast<const uint8_t*>(t->bitmap);
        b.t[0].values = static_cast<const uint8_t*>(t->values);
        b.t[0].dst = static_cast<uint8_t*>(wd);
        b.t[0].n = n;
        b.t[0].nnz = t->nnz;
        b.t[0].idx = idx;
        uint64_t sub_cap, blk_cap;
        batch_plan(b, &sub_cap, &blk_cap, count_ctas());
        b.tsub = L.tsub;
        b.blk = L.blk;
        b.hdr = L.hdr;
        if (aligned(t->bitmap, 16)) {
            CK(launch_count(b, S(stream)));  // no-op for an indexed tensor
            CK(launch_expand_tma(b, 2, S(stream)));
        } else {
            ScanArgs a = scan_args(t->bitmap, n, 0, n, L);
            a.check_total = 1;
            a.expect_total = t->nnz;
            if (idx) {
                a.cs = kSubElems;
                a.idx_in = idx;
            }
            ExpandArgs x = expand_args(t, n, 0, n, wd, L);
            a.tprefix = L.tprefix;
            CK(launch_scan(a, S(stream)));
            CK(launch_expand(x, 2, S(stream)));
        }
        idx = nullptr;
    } else if (!idx) {
        // rank table of the reference's decompress (codec.hpp:157-160): counts,
        // checks popcount == nnz and the padding bits, flat absolute offsets
        if (aligned(t->bitmap, 16)) {
            Batch b{};
            b.count = 1;
            b.check_total = 1;
            b.t[0].bitmap = static_cast<const uint8_t*>(t->bitmap);
            b.t[0].values = static_cast<const uint8_t*>(t->values);
            b.t[0].n = n;
            b.t[0].nnz = t->nnz;
            uint64_t sub_cap, blk_cap;
            batch_plan(b, &sub_cap, &blk_cap, count_ctas());
            b.tsub = L.tsub;
            b.blk = L.blk;
            b.hdr = L.hdr;
            CK(launch_count(b, S(stream)));
            CK(launch_flatten(L.tsub, L.blk + b.t[0].blk0, uint64_t(kCountSubs) * b.t[0].cbpc, ceil_div(n, kSubElems),
                              S(stream)));
        } else {
            ScanArgs a = scan_args(t->bitmap, n, 0, n, L);
            a.tsub = L.tsub;
            a.check_total = 1;
            a.expect_total = t->nnz;
            CK(launch_scan(a, S(stream)));
        }
        idx = L.tsub;
    }
    GemmLaunch g{};
    g.bitmap = static_cast<const uint8_t*>(t->bitmap);
    g.values = static_cast<const uint8_t*>(t->values);
    g.nnz = t->nnz;
    g.rows = t->rows;
    g.cols = t->cols;
    g.tokens = tokens;
    g.idx = idx;
    g.x = x_f16;
    g.x_ld = x_ld;
    g.part = reinterpret_cast<float*>(static_cast<char*>(ws) + L.bytes);
    g.y32 = y_f32;
    g.y16 = y_f16;
    g.hdr = L.hdr;
    g.w_dense = wd;
    CK(launch_gemm_fused(p, g, S(stream)));
    return ENDOR_OK;
}

// extract_rows / extract_cols (codec.hpp:239-297): validation of the index
// list (check_sorted_unique, codec.hpp:224-232), a count pass for ranks, then
// the gather.  Errors are device-latched (endor_cuda_sync_status).
static int extract_common(const endor_tensor_view* t, const uint64_t* sel, uint64_t nsel, void* out, void* ws,
                          size_t ws_bytes, void* stream, bool rows) {
    uint64_t n;
    int eb, st;
    if ((st = check_view(t, &n, &eb))) return st;
    if (nsel && (!sel || !out)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null index list or output");
    if (!aligned(out, eb)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "misaligned output");
    if (n && !aligned(t->bitmap, 16)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "extraction needs a 16-byte aligned bitmap");
    WsLayout L;
    if ((st = check_ws(ws, ws_bytes, n ? n : 1, &L))) return st;
    const auto* idx = reinterpret_cast<const unsigned long long*>(sel);
    CK(launch_validate_indices(idx, nsel, rows ? t->rows : t->cols, L.hdr, S(stream)));
    if (n == 0 || nsel == 0) return ENDOR_OK;
    Batch b{};
    b.count = 1;
    b.check_total = 1;
    b.t[0].bitmap = static_cast<const uint8_t*>(t->bitmap);
    b.t[0].values = static_cast<const uint8_t*>(t->values);
    b.t[0].n = n;
    b.t[0].nnz = t->nnz;
    uint64_t sub_cap, blk_cap;
    batch_plan(b, &sub_cap, &blk_cap, count_ctas());
    b.tsub = L.tsub;
    b.blk = L.blk;
    b.hdr = L.hdr;
    CK(launch_count(b, S(stream)));
    RankTable rt{};
    rt.bitmap = b.t[0].bitmap;
    rt.nbytes = (n + 7) / 8;
    rt.tsub = L.tsub + b.t[0].sub0;
    rt.blk = L.blk + b.t[0].blk0;
    rt.cbpc = b.t[0].cbpc;
    rt.ncta = b.t[0].ncta;
    rt.nsub = ceil_div(n, kSubElems);
    const auto* vals = static_cast<const uint8_t*>(t->values);
    if (rows && t->cols % kSubElems == 0 && aligned(out, 16)) {
        // rows start on sub-tile boundaries: the persistent TMA expand, tile t =
        // piece t % tpr of row sel[t / tpr], written to output row t / tpr
        b.t[0].dst = static_cast<uint8_t*>(out);
        b.sel = idx;
        b.rcols = t->cols;
        b.tpr = uint32_t(ceil_div(t->cols, kTileElems));
        b.ntiles = nsel * b.tpr;
        CK(launch_expand_tma_rows(b, eb, S(stream)));
    } else if (rows)
        CK(launch_extract_rows(rt, vals, t->nnz, t->cols, eb, idx, nsel, static_cast<uint8_t*>(out), L.hdr,
                               S(stream)));
    else
        CK(launch_extract_cols(rt, vals, t->nnz, t->rows, t->cols, eb, idx, nsel, static_cast<uint8_t*>(out),
                               L.hdr, S(stream)));
    return ENDOR_OK;
}

int endor_cuda_extract_rows(const endor_tensor_view* t, const uint64_t* rows_dev, uint64_t nsel, void* out,
                            void* ws, size_t ws_bytes, void* stream) {
    return extract_common(t, rows_dev, nsel, out, ws, ws_bytes, stream, true);
}

int endor_cuda_extract_cols(const endor_tensor_view* t, const uint64_t* cols_dev, uint64_t nsel, void* out,
                            void* ws, size_t ws_bytes, void* stream) {
    return extract_common(t, cols_dev, nsel, out, ws, ws_bytes, stream, false);
}

int endor_cuda_decompress_phase(const endor_tensor_view* t, void* dense_out, int phase, void* ws,
                                size_t ws_bytes, void* stream) {
    uint64_t n;
    int eb, st;
    if (phase != 1 && phase != 2) return fail(ENDOR_ERR_INVALID_ARGUMENT, "phase must be 1 or 2");
    if ((st = check_view(t, &n, &eb))) return st;
    if (n == 0) return ENDOR_OK;
    if (phase == 2 && (!dense_out || !aligned(dense_out, 16)))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "dense output must be non-null and 16-byte aligned");
    WsLayout L;
    if ((st = check_ws(ws, ws_bytes, n, &L))) return st;
    ScanArgs a = scan_args(t->bitmap, n, 0, n, L);
    a.check_total = 1;
    a.expect_total = t->nnz;
    return full_expand(t, n, eb, dense_out, L, a, S(stream), phase);
}

int endor_cuda_rank_index(const void* bitmap, uint64_t n, uint64_t chunk_size, uint64_t* prefix_out,
                          uint64_t* total_out, void* ws, size_t ws_bytes, void* stream) {
    if (!is_pow2_ge64(chunk_size))  // bitmap.hpp:118-120
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "chunk_size must be a power of two >= 64");
    if (n == 0) {
        if (total_out) CK(cudaMemsetAsync(total_out, 0, 8, S(stream)));
        return ENDOR_OK;
    }
    if (!bitmap || !aligned(bitmap, 4)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "bitmap must be non-null and 4-byte aligned");
    if (!prefix_out) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null prefix output");
    WsLayout L;
    int st;
    if ((st = check_ws(ws, ws_bytes, n, &L))) return st;
    ScanArgs a = scan_args(bitmap, n, 0, n, L);
    a.cs = chunk_size;
    a.idx_out = reinterpret_cast<unsigned long long*>(prefix_out);
    a.total_out = reinterpret_cast<unsigned long long*>(total_out);
    CK(launch_scan(a, S(stream)));
    return ENDOR_OK;
}

int endor_cuda_popcount(const void* bitmap, uint64_t n, uint64_t* total_out, void* ws,
                        size_t ws_bytes, void* stream) {
    if (!total_out) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null total output");
    if (n == 0) {
        CK(cudaMemsetAsync(total_out, 0, 8, S(stream)));
        return ENDOR_OK;
    }
    if (!bitmap || !aligned(bitmap, 4)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "bitmap must be non-null and 4-byte aligned");
    WsLayout L;
    int st;
    if ((st = check_ws(ws, ws_bytes, n, &L))) return st;
    ScanArgs a = scan_args(bitmap, n, 0, n, L);
    a.total_out = reinterpret_cast<unsigned long long*>(total_out);
    CK(launch_scan(a, S(stream)));
    return ENDOR_OK;
}

int endor_cuda_decompress_chunked(const endor_tensor_view* t, uint64_t cs, const uint64_t* prefix,
                                  uint64_t chunk_count, void* dense_out, void* ws, size_t ws_bytes,
                                  void* stream) {
    uint64_t n;
    int eb, st;
    if ((st = check_view(t, &n, &eb))) return st;
    // check_index (codec.hpp:170-176): the index must cover the bitmap; any
    // nonzero chunk size is a valid RankIndex (bitmap.hpp:104)
    const uint64_t chunks = (n == 0 || cs == 0) ? 0 : ceil_div(n, cs);
    if (cs == 0 || chunk_count != chunks) return fail(ENDOR_ERR_CORRUPTION, "rank index does not cover the bitmap");
    if (n == 0) return ENDOR_OK;
    if (!prefix) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null prefix");
    if (!dense_out || !aligned(dense_out, 16))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "dense output must be non-null and 16-byte aligned");
    WsLayout L;
    if ((st = check_ws(ws, ws_bytes, n, &L))) return st;
    const auto* idx = reinterpret_cast<const unsigned long long*>(prefix);
    if ((cs == uint64_t(kSubElems) || derive_chunk(cs)) && aligned(t->bitmap, 16) && aligned(prefix, 16)) {
        // fast path: the index supplies every sub-tile offset (chunk 1024), or
        // every chunk start with the producer deriving the sub-tile starts from
        // the staged bitmap (2048 / 4096 / 8192, checking every entry) -> one
        // expand launch, check_index's tail test inside it (codec.hpp:177-183)
        void* outs[1] = {dense_out};
        const uint64_t* pres[1] = {prefix};
        return endor_cuda_decompress_chunked_batch(t, pres, cs, outs, 1, ws, ws_bytes, stream);
    }
    if (aligned(t->bitmap, 16)) {
        // any other chunk size (the reference's default 4096, codec.hpp:19):
        // count the bitmap once (total == nnz covers the tail test), check every
        // index entry against the count tables, then the persistent TMA expand
        Batch b{};
        b.count = 1;
        b.check_total = 1;
        BatchTensor& T = b.t[0];
        T.bitmap = static_cast<const uint8_t*>(t->bitmap);
        T.values = static_cast<const uint8_t*>(t->values);
        T.dst = static_cast<uint8_t*>(dense_out);
        T.n = n;
        T.nnz = t->nnz;
        uint64_t sub_cap, blk_cap;
        batch_plan(b, &sub_cap, &blk_cap, count_ctas());  // within ws_layout(n)'s capacities
        b.tsub = L.tsub;
        b.blk = L.blk;
        b.hdr = L.hdr;
        CK(launch_count(b, S(stream)));
        CK(launch_verify_index(idx, chunks, cs, T.bitmap, n, b.tsub + T.sub0, b.blk + T.blk0,
                               uint64_t(kCountSubs) * T.cbpc, b.hdr, S(stream)));
        CK(launch_expand_tma(b, eb, S(stream)));
        return ENDOR_OK;
    }
    // bitmap not 16-byte aligned: general rank scan (tile offsets + flat
    // 1024-element sub-tile ranks, total == nnz), entry check, plain expand
    ScanArgs a = scan_args(t->bitmap, n, 0, n, L);
    a.check_total = 1;
    a.expect_total = t->nnz;
    a.tprefix = L.tprefix;
    a.tsub = L.tsub;
    CK(launch_scan(a, S(stream)));
    CK(launch_verify_index(idx, chunks, cs, static_cast<const uint8_t*>(t->bitmap), n, L.tsub, nullptr, 0, L.hdr,
                           S(stream)));
    CK(launch_expand(expand_args(t, n, 0, n, dense_out, L), eb, S(stream)));
    return ENDOR_OK;
}

int endor_cuda_decompress_chunked_batch(const endor_tensor_view* views, const uint64_t* const* prefixes,
                                        uint64_t cs, void* const* dense_outs, int count, void* ws,
                                        size_t ws_bytes, void* stream) {
    if (count < 0 || count > kMaxBatch || (count > 0 && (!views || !prefixes || !dense_outs)))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "batch must hold 0..64 tensors with prefixes and outputs");
    bool fast = cs == uint64_t(kSubElems) || derive_chunk(cs);
    for (int i = 0; i < count && fast; ++i) fast = aligned(views[i].bitmap, 16) && aligned(prefixes[i], 16);
    if (!fast) {  // general path, one tensor at a time (verifies every index entry)
        for (int i = 0; i < count; ++i) {
            uint64_t n = 0;
            int e = 0, st;
            if ((st = check_view(&views[i], &n, &e))) return st;
            const uint64_t chunks = (n == 0 || cs == 0) ? 0 : ceil_div(n, cs);
            if ((st = endor_cuda_decompress_chunked(&views[i], cs, prefixes[i], chunks, dense_outs[i], ws,
                                                    ws_bytes, stream)))
                return st;
        }
        return ENDOR_OK;
    }
    Batch b;
    int eb, st;
    uint64_t nmax;
    size_t need;
    if ((st = plan_batch(views, dense_outs, count, &b, &eb, &nmax, &need))) return st;
    // attach the indices (plan_batch drops empty tensors: walk both lists)
    for (int i = 0, j = 0; i < count; ++i) {
        if (views[i].rows * views[i].cols == 0) continue;
        if (!prefixes[i]) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null prefix");
        b.t[j].idx_subs = uint32_t(cs / kSubElems);
        b.t[j++].idx = reinterpret_cast<const unsigned long long*>(prefixes[i]);
    }
    if (b.count == 0) return ENDOR_OK;
    if (!ws || !aligned(ws, 256)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
    if (ws_bytes < sizeof(WsHeader)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "workspace too small");
    uint64_t sub_cap, blk_cap;
    batch_plan(b, &sub_cap, &blk_cap, count_ctas());
    b.check_total = 1;
    b.hdr = static_cast<WsHeader*>(ws);  // only the status word is used on this path
    b.tsub = nullptr;
    b.blk = nullptr;
    if (cs == uint64_t(kSubElems)) CK(launch_expand_tma(b, eb, S(stream)));
    else CK(launch_expand_tma_derive(b, eb, S(stream)));
    return ENDOR_OK;
}

// Range [b, e) of a tensor with its first value at *base_dev: scan (masking
// bits below b; b need not be word aligned) + the plain expand, writing
// exactly the elements of [b, e).  check: verify base + popcount == nnz.
static int range_expand(const endor_tensor_view* t, uint64_t n, int eb, uint64_t b, uint64_t e,
                        const unsigned long long* base_dev, bool check, void* dst, const WsLayout& L,
                        cudaStream_t s) {
    const uint64_t b0 = b & ~uint64_t(31);
    ScanArgs a = scan_args(t->bitmap, n, b0, e, L);
    a.lo = b;
    a.p0_ptr = base_dev;
    a.tprefix = dst ? L.tprefix : nullptr;
    if (check) {
        a.check_total = 1;
        a.expect_total = t->nnz;
    }
    CK(launch_scan(a, s));
    if (dst) {
        ExpandArgs x = expand_args(t, n, b0, e, dst, L);
        x.lo = b;
        CK(launch_expand(x, eb, s));
    }
    return ENDOR_OK;
}

int endor_cuda_decompress_chunk_into(const endor_tensor_view* t, uint64_t cs, const uint64_t* prefix,
                                     uint64_t chunk_count, uint64_t k, void* dense_out,
                                     uint64_t dense_out_bytes, void* ws, size_t ws_bytes,
                                     void* stream) {
    uint64_t n;
    int eb, st;
    if ((st = check_view(t, &n, &eb))) return st;
    const uint64_t chunks = (n == 0 || cs == 0) ? 0 : ceil_div(n, cs);
    if (cs == 0 || chunk_count != chunks) return fail(ENDOR_ERR_CORRUPTION, "rank index does not cover the bitmap");
    if (k >= chunk_count) return fail(ENDOR_ERR_BOUNDS, "chunk index out of range");  // codec.hpp:194
    if (dense_out_bytes != n * uint64_t(eb))  // codec.hpp:195-197
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "destination buffer must hold the full dense matrix");
    if (!prefix) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null prefix");
    if (!dense_out || !aligned(dense_out, 16))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "dense output must be non-null and 16-byte aligned");
    WsLayout L;
    if ((st = check_ws(ws, ws_bytes, n, &L))) return st;
    const auto* pre = reinterpret_cast<const unsigned long long*>(prefix);
    const uint64_t last = chunk_count - 1;  // chunk_count >= 1 here (k < chunk_count)
    // check_index tail (codec.hpp:177-183): prefix[last] + popcount(last chunk) == nnz
    if (k != last && (st = range_expand(t, n, eb, last * cs, n, pre + last, true, nullptr, L, S(stream))))
        return st;
    const uint64_t b = k * cs, e = (b + cs < n) ? b + cs : n;
    return range_expand(t, n, eb, b, e, pre + k, k == last, dense_out, L, S(stream));
}

int endor_cuda_compress(uint64_t rows, uint64_t cols, int32_t dtype, const void* dense,
                        void* bitmap_out, void* values_out, uint64_t* nnz_out_host,
                        int32_t* negzero_out_host, void* ws, size_t ws_bytes, void* stream) {
    uint64_t n;
    const int eb = eb_of(dtype);
    if (!eb) return fail(ENDOR_ERR_INVALID_ARGUMENT, "unknown dtype code");
    if (!checked_n(rows, cols, &n)) return fail(ENDOR_ERR_SIZE, "matrix dimensions overflow the addressable element count");
    if (!nnz_out_host) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null nnz output");
    if (n == 0) {
        *nnz_out_host = 0;
        if (negzero_out_host) *negzero_out_host = 0;
        return ENDOR_OK;
    }
    if (!dense || !bitmap_out || !values_out) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null buffer");
    if (!aligned(bitmap_out, 4) || !aligned(dense, eb)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "misaligned buffer");
    WsLayout L;
    int st;
    if ((st = check_ws(ws, ws_bytes, n, &L))) return st;
    CK(cudaMemsetAsync(&L.hdr->aux[2], 0, 8, S(stream)));
    CK(launch_bitmap(dense, n, eb, bitmap_out, L, S(stream)));
    ScanArgs a = scan_args(bitmap_out, n, 0, n, L);
    a.tprefix = L.tprefix;
    CK(launch_scan(a, S(stream)));
    CK(launch_compact(dense, n, eb, bitmap_out, L, values_out, S(stream)));
    unsigned long long hv[2];
    CK(cudaMemcpyAsync(&hv[0], &L.hdr->total, 8, cudaMemcpyDeviceToHost, S(stream)));
    CK(cudaMemcpyAsync(&hv[1], &L.hdr->aux[2], 8, cudaMemcpyDeviceToHost, S(stream)));
    CK(cudaStreamSynchronize(S(stream)));
    *nnz_out_host = hv[0];
    if (negzero_out_host) *negzero_out_host = hv[1] ? 1 : 0;
    return endor_cuda_sync_status(ws, stream);
}

int endor_cuda_quantize_values(const void* values_f16, uint64_t nnz, void* q_out, float* scale_out_host,
                               void* ws, size_t ws_bytes, void* stream) {
    if (!scale_out_host) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null scale output");
    if (nnz && (!values_f16 || !q_out || !aligned(values_f16, 2)))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "null or misaligned buffer");
    WsLayout L;
    int st;
    if ((st = check_ws(ws, ws_bytes, 1, &L))) return st;
    float* scale_dev = reinterpret_cast<float*>(&L.hdr->aux[3]);
    unsigned int* amax = reinterpret_cast<unsigned int*>(&L.hdr->aux[3]) + 1;
    CK(launch_quantize(values_f16, nnz, q_out, scale_dev, amax, S(stream)));
    CK(cudaMemcpyAsync(scale_out_host, scale_dev, sizeof(float), cudaMemcpyDeviceToHost, S(stream)));
    CK(cudaStreamSynchronize(S(stream)));
    return ENDOR_OK;
}

int endor_cuda_dequantize_values(const void* q_i8, uint64_t nnz, float scale, void* out_f16, void* stream) {
    if (nnz && (!q_i8 || !out_f16 || !aligned(out_f16, 2))) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null or misaligned buffer");
    CK(launch_dequant_values(q_i8, nnz, scale, out_f16, S(stream)));
    return ENDOR_OK;
}

int endor_cuda_synth_weight(uint64_t rows, uint64_t cols, int32_t dtype, uint64_t seed,
                            uint64_t row0, uint64_t nrows, void* out, void* stream) {
    uint64_t n;
    const int eb = eb_of(dtype);
    if (!eb) return fail(ENDOR_ERR_INVALID_ARGUMENT, "unknown dtype code");
    if (!checked_n(rows, cols, &n)) return fail(ENDOR_ERR_SIZE, "matrix dimensions overflow the addressable element count");
    if (row0 > rows || nrows > rows - row0) return fail(ENDOR_ERR_BOUNDS, "row range outside the matrix");
    if (nrows == 0 || cols == 0) return ENDOR_OK;
    if (!out || !aligned(out, eb)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null or misaligned output");
    CK(launch_synth(row0 * cols, nrows * cols, eb, seed, out, S(stream)));
    return ENDOR_OK;
}

int endor_cuda_magnitude_prune(uint64_t n, int32_t dtype, double sparsity, void* w, void* ws,
                               size_t ws_bytes, void* stream) {
    const int eb = eb_of(dtype);
    if (!eb) return fail(ENDOR_ERR_INVALID_ARGUMENT, "unknown dtype code");
    if (!(sparsity >= 0.0 && sparsity < 1.0))  // weight_gen.hpp:97-99
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "sparsity must be in [0, 1)");
    const uint64_t target = uint64_t(sparsity * double(n));  // weight_gen.hpp:102
    if (target == 0) return ENDOR_OK;
    if (!w || !aligned(w, eb)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null or misaligned weights");
    WsLayout L;
    int st;
    if ((st = check_ws(ws, ws_bytes, n, &L))) return st;
    CK(launch_prune(static_cast<uint8_t*>(w), n, eb, target, L, S(stream)));
    return ENDOR_OK;
}

int endor_cuda_gemv(uint64_t rows, uint64_t cols, const void* w_f16, const void* x_f16, float* y_f32,
                    void* y_f16, void* stream) {
    uint64_t n;
    if (!checked_n(rows, cols, &n)) return fail(ENDOR_ERR_SIZE, "matrix dimensions overflow the addressable element count");
    if (rows == 0) return ENDOR_OK;
    if ((cols > 0 && (!w_f16 || !x_f16)) || (!y_f32 && !y_f16))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "null buffer");
    if (!aligned(w_f16, 2) || !aligned(x_f16, 2)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "misaligned f16 buffer");
    CK(launch_gemv(rows, cols, w_f16, x_f16, y_f32, y_f16, S(stream)));
    return ENDOR_OK;
}

int endor_cuda_gemv_batch(const uint64_t* rows, const uint64_t* cols, const void* const* w_f16,
                          const void* const* x_f16, float* const* y_f32, void* const* y_f16, int count,
                          void* stream) {
    if (count < 0 || count > kMaxBatch || (count > 0 && (!rows || !cols || !w_f16 || !x_f16)))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "batch must hold 0..64 GEMVs");
    GemvBatch gb{};
    for (int i = 0; i < count; ++i) {
        uint64_t n;
        if (!checked_n(rows[i], cols[i], &n))
            return fail(ENDOR_ERR_SIZE, "matrix dimensions overflow the addressable element count");
        float* y32 = y_f32 ? y_f32[i] : nullptr;
        void* y16 = y_f16 ? y_f16[i] : nullptr;
        if (rows[i] == 0) continue;
        if ((cols[i] > 0 && (!w_f16[i] || !x_f16[i])) || (!y32 && !y16))
            return fail(ENDOR_ERR_INVALID_ARGUMENT, "null buffer");
        if (cols[i] % 8 || !aligned(w_f16[i], 16) || !aligned(x_f16[i], 16)) {
            // outside the vector layout: run it alone on the generic kernel
            if (!aligned(w_f16[i], 2) || !aligned(x_f16[i], 2))
                return fail(ENDOR_ERR_INVALID_ARGUMENT, "misaligned f16 buffer");
            CK(launch_gemv(rows[i], cols[i], w_f16[i], x_f16[i], y32, y16, S(stream)));
            continue;
        }
        gb.rows[gb.count] = rows[i];
        gb.cols[gb.count] = cols[i];
        gb.w[gb.count] = w_f16[i];
        gb.x[gb.count] = x_f16[i];
        gb.y32[gb.count] = y32;
        gb.y16[gb.count] = y16;
        ++gb.count;
    }
    if (gb.count) CK(launch_gemv_batch(gb, S(stream)));
    return ENDOR_OK;
}

// ---- host-buffer convenience (sync) --------------------------------------------
namespace {
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t need(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    ~DevBuf() { cudaFree(p); }
};

// Grow-only pinned host staging buffer.
struct PinBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t need(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocDefault);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    ~PinBuf() { cudaFreeHost(p); }
};

// Grow-only device buffers reused by the synchronous host-buffer entry points
// (one set per host thread and device).
struct HostSession {
    int device = -1;
    DevBuf bm, vals, dense, ws, prefix;
    PinBuf pin_in, pin_out;  // chunk_into staging: one DMA each way
    cudaStream_t stream = nullptr;  // non-blocking, so host threads fanning out calls overlap
    ~HostSession() {
        if (stream) cudaStreamDestroy(stream);
    }
};
// owned per thread: a thread's buffers and stream are released when it exits
// (callers may fan chunk calls out over short-lived threads)
thread_local std::unique_ptr<HostSession> g_sess;

int session(HostSession** out, uint64_t n) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (!g_sess || g_sess->device != dev) {
        g_sess = std::make_unique<HostSession>();
        g_sess->device = dev;
    }
    const size_t wsb = ws_layout(nullptr, n).bytes;
    if (wsb > g_sess->ws.cap) {
        CK(g_sess->ws.need(wsb));
        CK(cudaMemset(g_sess->ws.p, 0, g_sess->ws.cap));
    }
    *out = g_sess.get();
    return ENDOR_OK;
}

// Validate + upload a host tensor; fills the device view.
int upload(HostSession* s, uint64_t rows, uint64_t cols, int32_t dtype, const void* bitmap_host,
           const void* values_host, uint64_t nnz, endor_tensor_view* v, uint64_t* n_out) {
    uint64_t n;
    const int eb = eb_of(dtype);
    if (!eb) return fail(ENDOR_ERR_INVALID_ARGUMENT, "unknown dtype code");
    if (!checked_n(rows, cols, &n)) return fail(ENDOR_ERR_SIZE, "matrix dimensions overflow the addressable element count");
    if (nnz > n) return fail(ENDOR_ERR_CORRUPTION, "values length does not match bitmap popcount");
    const size_t bmb = (n + 7) / 8, vb = nnz * eb;
    CK(s->bm.need(bmb + 16));
    CK(s->vals.need(vb + 16));
    if (bmb) CK(cudaMemcpy(s->bm.p, bitmap_host, bmb, cudaMemcpyHostToDevice));
    if (vb) CK(cudaMemcpy(s->vals.p, values_host, vb, cudaMemcpyHostToDevice));
    *v = endor_tensor_view{rows, cols, dtype, 0, s->bm.p, s->vals.p, nnz};
    *n_out = n;
    return ENDOR_OK;
}
}  // namespace

#define ST(expr)                   \
    do {                           \
        int st_ = (expr);          \
        if (st_) return st_;       \
    } while (0)

int endor_cuda_decompress_host(uint64_t rows, uint64_t cols, int32_t dtype, const void* bitmap_host,
                               const void* values_host, uint64_t nnz, void* dense_host_out) {
    HostSession* s;
    endor_tensor_view v;
    uint64_t n;
    ST(session(&s, 1));
    ST(upload(s, rows, cols, dtype, bitmap_host, values_host, nnz, &v, &n));
    if (n == 0) return ENDOR_OK;
    ST(session(&s, n));
    const size_t db = n * eb_of(dtype);
    CK(s->dense.need(db + 16));
    ST(endor_cuda_decompress(&v, s->dense.p, s->ws.p, s->ws.cap, nullptr));
    ST(endor_cuda_sync_status(s->ws.p, nullptr));
    CK(cudaMemcpy(dense_host_out, s->dense.p, db, cudaMemcpyDeviceToHost));
    return ENDOR_OK;
}

int endor_cuda_rank_index_host(const void* bitmap_host, uint64_t n, uint64_t chunk_size,
                               uint64_t* prefix_host_out) {
    if (!is_pow2_ge64(chunk_size))
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "chunk_size must be a power of two >= 64");
    if (n == 0) return ENDOR_OK;
    HostSession* s;
    ST(session(&s, n));
    const size_t bmb = (n + 7) / 8, chunks = ceil_div(n, chunk_size);
    CK(s->bm.need(bmb + 16));
    CK(s->prefix.need(chunks * 8));
    CK(cudaMemcpy(s->bm.p, bitmap_host, bmb, cudaMemcpyHostToDevice));
    ST(endor_cuda_rank_index(s->bm.p, n, chunk_size, static_cast<uint64_t*>(s->prefix.p), nullptr,
                             s->ws.p, s->ws.cap, nullptr));
    ST(endor_cuda_sync_status(s->ws.p, nullptr));
    CK(cudaMemcpy(prefix_host_out, s->prefix.p, chunks * 8, cudaMemcpyDeviceToHost));
    return ENDOR_OK;
}

int endor_cuda_decompress_chunked_host(uint64_t rows, uint64_t cols, int32_t dtype,
                                       const void* bitmap_host, const void* values_host,
                                       uint64_t nnz, uint64_t chunk_size,
                                       const uint64_t* prefix_host, uint64_t chunk_count,
                                       void* dense_host_out) {
    HostSession* s;
    endor_tensor_view v;
    uint64_t n;
    ST(session(&s, 1));
    ST(upload(s, rows, cols, dtype, bitmap_host, values_host, nnz, &v, &n));
    ST(session(&s, n));
    CK(s->prefix.need(chunk_count * 8 + 8));
    if (chunk_count) CK(cudaMemcpy(s->prefix.p, prefix_host, chunk_count * 8, cudaMemcpyHostToDevice));
    const size_t db = n * eb_of(dtype);
    CK(s->dense.need(db + 16));
    ST(endor_cuda_decompress_chunked(&v, chunk_size, static_cast<const uint64_t*>(s->prefix.p),
                                     chunk_count, s->dense.p, s->ws.p, s->ws.cap, nullptr));
    ST(endor_cuda_sync_status(s->ws.p, nullptr));
    if (db) CK(cudaMemcpy(dense_host_out, s->dense.p, db, cudaMemcpyDeviceToHost));
    return ENDOR_OK;
}

int endor_cuda_decompress_chunk_into_host(uint64_t rows, uint64_t cols, int32_t dtype,
                                          const void* bitmap_host, const void* values_host,
                                          uint64_t nnz, uint64_t cs, const uint64_t* prefix_host,
                                          uint64_t chunk_count, uint64_t k, void* dense_host,
                                          uint64_t dense_host_bytes) {
    // Moves only what chunk k needs -- the last chunk's bitmap bytes for the
    // check_index tail, chunk k's bitmap bytes and at most one chunk of values
    // from prefix[k] -- gathered into a pinned staging buffer and sent as ONE
    // DMA, and returns chunk k's dense bytes through one pinned DMA, so a
    // caller fanning decompress_chunk_into out over the chunks from several
    // host threads (the reference's pattern, codec.hpp:203-204) pays per chunk,
    // not per tensor, and the threads' host-side copies run in parallel (each
    // thread has its own session and non-blocking stream).  Each range runs as
    // its own sub-tensor view starting at the 32-bit word holding its first bit.
    uint64_t n;
    const int eb = eb_of(dtype);
    if (!eb) return fail(ENDOR_ERR_INVALID_ARGUMENT, "unknown dtype code");
    if (!checked_n(rows, cols, &n)) return fail(ENDOR_ERR_SIZE, "matrix dimensions overflow the addressable element count");
    if (nnz > n) return fail(ENDOR_ERR_CORRUPTION, "values length does not match bitmap popcount");
    // check_index first (codec.hpp:193), exactly as the reference orders it
    const uint64_t chunks = (n == 0 || cs == 0) ? 0 : ceil_div(n, cs);
    if (cs == 0 || chunk_count != chunks) return fail(ENDOR_ERR_CORRUPTION, "rank index does not cover the bitmap");
    if (chunk_count == 0) return fail(ENDOR_ERR_BOUNDS, "chunk index out of range");  // codec.hpp:177,194
    if (!prefix_host || !bitmap_host) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null prefix or bitmap");
    const uint64_t last = chunk_count - 1;
    const uint64_t lb = last * cs, lb0 = lb & ~uint64_t(31), nt = n - lb0;  // tail view: bits [lb0, n)
    const bool go = k < chunk_count && dense_host_bytes == n * uint64_t(eb);
    const uint64_t b = go ? k * cs : 0, e = go ? ((b + cs < n) ? b + cs : n) : 0;
    // chunk view: bits [b0, e) of a view whose length runs to the next 32-bit
    // word boundary (or the tensor's end), so the bits after e in its last
    // bytes belong to the view, not to its padding
    const uint64_t b0 = b & ~uint64_t(31);
    const uint64_t nc = ((e + 31) & ~uint64_t(31)) < n ? ((e + 31) & ~uint64_t(31)) - b0 : n - b0;
    const uint64_t p = go ? prefix_host[k] : 0;
    const uint64_t w = go && p <= nnz ? ((e - b < nnz - p) ? e - b : nnz - p) : 0;  // values moved
    if (go && p > nnz) return fail(ENDOR_ERR_CORRUPTION, "rank index entry beyond the values");
    if (go && ((w && !values_host) || !dense_host)) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null buffer");
    HostSession* s;
    ST(session(&s, nt > nc ? nt : nc));
    if (!s->stream) CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    cudaStream_t st = s->stream;
    const WsLayout L = ws_layout(s->ws.p, nt > nc ? nt : nc);
    // one staging image, host and device alike: [prefix[last], 0][tail bitmap][chunk bitmap][values]
    auto up16 = [](size_t x) { return (x + 15) & ~size_t(15); };
    const size_t tbm = (nt + 7) / 8, cbm = go ? (nc + 7) / 8 : 0, vb = w * eb;
    const size_t o_tail = 16, o_chunk = o_tail + up16(tbm), o_vals = o_chunk + up16(cbm), in_bytes = o_vals + vb;
    CK(s->pin_in.need(in_bytes + 16));
    CK(s->bm.need(in_bytes + 16));
    uint8_t* hin = static_cast<uint8_t*>(s->pin_in.p);
    uint8_t* din = static_cast<uint8_t*>(s->bm.p);
    const unsigned long long pair[2] = {prefix_host[last], 0ull};  // tail base, chunk base (view-relative)
    memcpy(hin, pair, 16);
    memcpy(hin + o_tail, static_cast<const uint8_t*>(bitmap_host) + lb0 / 8, tbm);
    if (go) {
        memcpy(hin + o_chunk, static_cast<const uint8_t*>(bitmap_host) + b0 / 8, cbm);
        if (vb) memcpy(hin + o_vals, static_cast<const uint8_t*>(values_host) + p * eb, vb);
    }
    CK(cudaMemcpyAsync(din, hin, go ? in_bytes : o_chunk, cudaMemcpyHostToDevice, st));
    auto* pre = reinterpret_cast<const unsigned long long*>(din);
    // the tail test: prefix[last] + popcount(bits [lb, n)) == nnz
    endor_tensor_view tv{1, nt, dtype, 0, din + o_tail, nullptr, nnz};
    ST(range_expand(&tv, nt, eb, lb - lb0, nt, pre, true, nullptr, L, st));
    if (!go) {  // the tail's CORRUPTION outranks BOUNDS / INVALID (codec.hpp:193-197)
        ST(endor_cuda_sync_status(s->ws.p, st));
        if (k >= chunk_count) return fail(ENDOR_ERR_BOUNDS, "chunk index out of range");
        return fail(ENDOR_ERR_INVALID_ARGUMENT, "destination buffer must hold the full dense matrix");
    }
    CK(s->dense.need(nc * eb + 16));
    // chunk k's values start at view rank 0 of the window; running past it is CORRUPTION
    endor_tensor_view cv{1, nc, dtype, 0, din + o_chunk, din + o_vals, w};
    ST(range_expand(&cv, nc, eb, b - b0, e - b0, pre + 1, false, s->dense.p, L, st));
    const size_t ob = (e - b) * eb;
    CK(s->pin_out.need(ob + 16));
    uint8_t* hout = static_cast<uint8_t*>(s->pin_out.p);
    CK(cudaMemcpyAsync(hout + 8, static_cast<uint8_t*>(s->dense.p) + (b - b0) * eb, ob, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hout, &L.hdr->status, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    uint32_t status;
    memcpy(&status, hout, 4);
    if (status) return endor_cuda_sync_status(s->ws.p, st);  // reports and resets it
    memcpy(static_cast<uint8_t*>(dense_host) + b * eb, hout + 8, ob);
    return ENDOR_OK;
}

int endor_cuda_compress_host(uint64_t rows, uint64_t cols, int32_t dtype, const void* dense_host,
                             void* bitmap_host_out, void* values_host_out, uint64_t* nnz_out,
                             int32_t* negzero_out) {
    uint64_t n;
    const int eb = eb_of(dtype);
    if (!eb) return fail(ENDOR_ERR_INVALID_ARGUMENT, "unknown dtype code");
    if (!checked_n(rows, cols, &n)) return fail(ENDOR_ERR_SIZE, "matrix dimensions overflow the addressable element count");
    if (!nnz_out) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null nnz output");
    if (n == 0) {
        *nnz_out = 0;
        if (negzero_out) *negzero_out = 0;
        return ENDOR_OK;
    }
    HostSession* s;
    ST(session(&s, n));
    const size_t bmb = (n + 7) / 8, db = n * eb;
    CK(s->dense.need(db + 16));
    CK(s->bm.need(bmb + 16));
    CK(s->vals.need(db + 16));
    CK(cudaMemcpy(s->dense.p, dense_host, db, cudaMemcpyHostToDevice));
    ST(endor_cuda_compress(rows, cols, dtype, s->dense.p, s->bm.p, s->vals.p, nnz_out, negzero_out,
                           s->ws.p, s->ws.cap, nullptr));
    CK(cudaMemcpy(bitmap_host_out, s->bm.p, bmb, cudaMemcpyDeviceToHost));
    if (*nnz_out) CK(cudaMemcpy(values_host_out, s->vals.p, *nnz_out * eb, cudaMemcpyDeviceToHost));
    return ENDOR_OK;
}

// extract_rows / extract_cols (codec.hpp:239-297) on host buffers: index
// validation order and exceptions as check_sorted_unique (codec.hpp:224-232).
static int extract_host(uint64_t rows, uint64_t cols, int32_t dtype, const void* bitmap_host,
                        const void* values_host, uint64_t nnz, const uint64_t* sel_host, uint64_t nsel,
                        void* out_host, bool by_rows) {
    HostSession* s;
    endor_tensor_view v;
    uint64_t n;
    ST(session(&s, 1));
    ST(upload(s, rows, cols, dtype, bitmap_host, values_host, nnz, &v, &n));
    ST(session(&s, n ? n : 1));
    const uint64_t out_elems = by_rows ? nsel * cols : rows * nsel;
    const size_t ob = out_elems * eb_of(dtype);
    if (nsel && !sel_host) return fail(ENDOR_ERR_INVALID_ARGUMENT, "null index list");
    CK(s->prefix.need(nsel * 8 + 16));
    CK(s->dense.need(ob + 16));
    if (nsel) CK(cudaMemcpy(s->prefix.p, sel_host, nsel * 8, cudaMemcpyHostToDevice));
    ST((by_rows ? endor_cuda_extract_rows : endor_cuda_extract_cols)(&v, static_cast<const uint64_t*>(s->prefix.p),
                                                                      nsel, s->dense.p, s->ws.p, s->ws.cap, nullptr));
    ST(endor_cuda_sync_status(s->ws.p, nullptr));
    if (ob) CK(cudaMemcpy(out_host, s->dense.p, ob, cudaMemcpyDeviceToHost));
    return ENDOR_OK;
}

int endor_cuda_extract_rows_host(uint64_t rows, uint64_t cols, int32_t dtype, const void* bitmap_host,
                                 const void* values_host, uint64_t nnz, const uint64_t* rows_host, uint64_t nsel,
                                 void* out_host) {
    return extract_host(rows, cols, dtype, bitmap_host, values_host, nnz, rows_host, nsel, out_host, true);
}

int endor_cuda_extract_cols_host(uint64_t rows, uint64_t cols, int32_t dtype, const void* bitmap_host,
                                 const void* values_host, uint64_t nnz, const uint64_t* cols_host, uint64_t nsel,
                                 void* out_host) {
    return extract_host(rows, cols, dtype, bitmap_host, values_host, nnz, cols_host, nsel, out_host, false);
}

int endor_cuda_quantize_values_host(const void* values_f16_host, uint64_t nnz, void* q_host_out,
                                    float* scale_out) {
    HostSession* s;
    ST(session(&s, 1));
    CK(s->vals.need(nnz * 2 + 16));
    CK(s->dense.need(nnz + 16));
    if (nnz) CK(cudaMemcpy(s->vals.p, values_f16_host, nnz * 2, cudaMemcpyHostToDevice));
    ST(endor_cuda_quantize_values(s->vals.p, nnz, s->dense.p, scale_out, s->ws.p, s->ws.cap, nullptr));
    if (nnz) CK(cudaMemcpy(q_host_out, s->dense.p, nnz, cudaMemcpyDeviceToHost));
    return ENDOR_OK;
}

int endor_cuda_dequantize_values_host(const void* q_host, uint64_t nnz, float scale, void* f16_host_out) {
    HostSession* s;
    ST(session(&s, 1));
    CK(s->vals.need(nnz + 16));
    CK(s->dense.need(nnz * 2 + 16));
    if (nnz) CK(cudaMemcpy(s->vals.p, q_host, nnz, cudaMemcpyHostToDevice));
    ST(endor_cuda_dequantize_values(s->vals.p, nnz, scale, s->dense.p, nullptr));
    if (nnz) CK(cudaMemcpy(f16_host_out, s->dense.p, nnz * 2, cudaMemcpyDeviceToHost));
    return ENDOR_OK;
}

void* endor_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
        g_last_error = "cudaHostAlloc failed";
        return nullptr;
    }
    return p;
}

void endor_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

}  // extern "C"
