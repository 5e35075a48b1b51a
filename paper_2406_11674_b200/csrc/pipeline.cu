// pipeline.cu -- the Endor offload pipeline, executed for real.
//
// The reference only models these stages analytically, one after another
// with no overlap (Endor mode: CpuToGpu c*B/bw -> Decompress -> Compute,
// sim.hpp:200-204; overlap deliberately not modelled, sim.hpp:122-124).
// Here each op's compressed bytes (bitmap + values, PCIe-side traffic =
// compression_ratio x dense, codec.hpp:75-80) stream from pinned host memory
// on a dedicated copy stream into a ring of device staging slots; the compute
// stream waits on the slot's copy event, runs scan + expand + GEMV, and
// releases the slot, so H2D of op i+1.. overlaps decompress+GEMV of op i.
// When the caller only wants y = W x (no dense_dev), the op runs as one fused
// decompress -> GEMV (gemv_fused.cu): the dense W never touches HBM.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys / ncu timelines
#include <stdint.h>

#include <new>
#include <string>
#include <vector>

#include "common.cuh"
#include "endor_cuda.h"
#include "kernels.h"

using namespace endor_b200;

struct endor_pipeline {
    int device = 0;
    int depth = 2;
    uint64_t max_elems = 0;
    cudaStream_t copy = nullptr, compute = nullptr;
    struct Slot {
        uint8_t* bitmap = nullptr;  // ceil(max/8) rounded up
        uint8_t* values = nullptr;  // max*2 bytes
        uint64_t* prefix = nullptr; // ceil(max/1024) u64: the op's optional RankIndex at chunk 1024
        uint8_t* coded = nullptr;   // coded-values blob (vcode.cu), allocated on the first coded op
        cudaEvent_t free_ev = nullptr;
    };
    std::vector<Slot> slots;
    uint8_t* dense[2] = {nullptr, nullptr};
    void* ws = nullptr;
    size_t ws_bytes = 0;
    // per-op timing events (grown on demand)
    std::vector<cudaEvent_t> h2d_beg, h2d_end, dec_beg, dec_end, op_end;
    endor_reader* reader = nullptr;  // file-sourced ops (created on first use)
    int last_nops = 0;
    uint64_t last_h2d_bytes = 0, last_dense_bytes = 0, last_launches = 0;
};

namespace {
// CUDA and argument errors go through the C ABI's last-error slot
// (endor_cuda_last_error_string), like every other entry point
int perr(cudaError_t e, const char* where) {
    return set_last_error(ENDOR_ERR_CUDA, (std::string(where) + ": " + cudaGetErrorString(e)).c_str());
}
int pbad(const char* what) { return set_last_error(ENDOR_ERR_INVALID_ARGUMENT, what); }
#define PK(expr)                                             \
    do {                                                     \
        cudaError_t e_ = (expr);                             \
        if (e_ != cudaSuccess) return perr(e_, #expr);       \
    } while (0)

int ensure_events(endor_pipeline* p, int nops) {
    auto grow = [&](std::vector<cudaEvent_t>& v) -> cudaError_t {
        while (int(v.size()) < nops) {
            cudaEvent_t e;
            cudaError_t r = cudaEventCreate(&e);
            if (r != cudaSuccess) return r;
            v.push_back(e);
        }
        return cudaSuccess;
    };
    PK(grow(p->h2d_beg));
    PK(grow(p->h2d_end));
    PK(grow(p->dec_beg));
    PK(grow(p->dec_end));
    PK(grow(p->op_end));
    return ENDOR_OK;
}
}  // namespace

extern "C" {

int endor_pipeline_create(int device_ordinal, uint64_t max_op_elems, int ring_depth,
                          endor_pipeline** out) {
    if (!out || max_op_elems == 0) return pbad("null output or zero max_op_elems");
    auto* p = new (std::nothrow) endor_pipeline();
    if (!p) return ENDOR_ERR_CUDA;
    p->device = device_ordinal;
    p->depth = ring_depth < 2 ? 2 : ring_depth;
    p->max_elems = max_op_elems;
    PK(cudaSetDevice(device_ordinal));
    PK(cudaStreamCreateWithFlags(&p->copy, cudaStreamNonBlocking));
    PK(cudaStreamCreateWithFlags(&p->compute, cudaStreamNonBlocking));
    const size_t bmb = align256((max_op_elems + 7) / 8 + 16);
    const size_t vb = align256(max_op_elems * 2 + 16);
    p->slots.resize(p->depth);
    for (auto& s : p->slots) {
        PK(cudaMalloc(&s.bitmap, bmb));
        PK(cudaMalloc(&s.values, vb));
        PK(cudaMalloc(&s.prefix, align256((max_op_elems + 1023) / 1024 * 8 + 8)));
        PK(cudaEventCreateWithFlags(&s.free_ev, cudaEventDisableTiming));
        PK(cudaEventRecord(s.free_ev, p->compute));
    }
    for (auto& d : p->dense) PK(cudaMalloc(&d, align256(max_op_elems * 2)));
    p->ws_bytes = endor_cuda_workspace_bytes(max_op_elems, 1);
    PK(cudaMalloc(&p->ws, p->ws_bytes));
    PK(cudaMemsetAsync(p->ws, 0, p->ws_bytes, p->compute));
    PK(cudaStreamSynchronize(p->compute));
    *out = p;
    return ENDOR_OK;
}

int endor_pipeline_destroy(endor_pipeline* p) {
    if (!p) return ENDOR_OK;
    cudaSetDevice(p->device);
    cudaStreamSynchronize(p->copy);
    cudaStreamSynchronize(p->compute);
    for (auto& s : p->slots) {
        cudaFree(s.bitmap);
        cudaFree(s.values);
        cudaFree(s.prefix);
        cudaFree(s.coded);
        cudaEventDestroy(s.free_ev);
    }
    for (auto& d : p->dense) cudaFree(d);
    cudaFree(p->ws);
    endor_reader_destroy(p->reader);
    for (auto* v : {&p->h2d_beg, &p->h2d_end, &p->dec_beg, &p->dec_end, &p->op_end})
        for (auto e : *v) cudaEventDestroy(e);
    cudaStreamDestroy(p->copy);
    cudaStreamDestroy(p->compute);
    delete p;
    return ENDOR_OK;
}

void* endor_pipeline_stream(endor_pipeline* p) { return p ? p->compute : nullptr; }

namespace {
// NVTX range for the enqueue of one pipeline stage (no-ops without a tool attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

int endor_pipeline_run(endor_pipeline* p, const endor_pipeline_op* ops, int nops, int sync) {
    if (!p || (nops > 0 && !ops)) return pbad("null pipeline or ops");
    NvtxRange run_range("endor_pipeline_run");
    PK(cudaSetDevice(p->device));
    int st = ensure_events(p, nops);
    if (st) return st;
    // GEMM ops (tokens > 1) need split-K partials (and, past the two-pass
    // threshold, a dense W) in the workspace: grow it once, before enqueueing
    size_t need = p->ws_bytes;
    for (int i = 0; i < nops; ++i)
        if (ops[i].tokens > 1) {
            const size_t b = endor_cuda_gemm_workspace_bytes(ops[i].rows, ops[i].cols, ops[i].tokens);
            need = b > need ? b : need;
        }
    if (need > p->ws_bytes) {
        PK(cudaStreamSynchronize(p->compute));
        PK(cudaFree(p->ws));
        p->ws = nullptr;
        PK(cudaMalloc(&p->ws, need));
        p->ws_bytes = need;
        PK(cudaMemsetAsync(p->ws, 0, need, p->compute));
    }
    uint64_t h2d = 0, dense = 0, launches = 0;
    for (int i = 0; i < nops; ++i) {
        const endor_pipeline_op& op = ops[i];
        const uint64_t n = op.rows * op.cols;
        const int eb = op.dtype == ENDOR_DTYPE_F16 ? 2 : 1;     // packed-value bytes (H2D)
        const bool deq = (op.flags & 1) != 0;                    // i8 values -> f16 W
        const int ob = (op.dtype == ENDOR_DTYPE_F16 || deq) ? 2 : 1;  // dense bytes
        if (op.rows && op.cols > UINT64_MAX / op.rows)
            return set_last_error(ENDOR_ERR_SIZE, "matrix dimensions overflow the addressable element count");
        if (n > p->max_elems) return pbad("op larger than the pipeline's max_op_elems");
        if ((op.dtype != ENDOR_DTYPE_F16 && op.dtype != ENDOR_DTYPE_I8) || (deq && op.dtype != ENDOR_DTYPE_I8))
            return pbad("unknown dtype, or dequant flag on a non-i8 op");
        // values length vs bitmap size (codec.hpp:34-39) BEFORE any copy is
        // enqueued: the staging slot holds at most max_op_elems values
        if (op.nnz > n) return set_last_error(ENDOR_ERR_CORRUPTION, "values length does not match bitmap popcount");
        if ((op.x_dev || op.y_dev) && ob != 2) return pbad("GEMV ops need an f16 (or dequantized) W");
        const bool gemm = op.tokens > 1 && op.x_dev && op.y_dev;
        if (gemm && (deq || op.dtype != ENDOR_DTYPE_F16 || op.cols % 8 || op.dense_dev))
            return pbad("GEMM ops need an f16 W with cols % 8 == 0 and no dense_dev");
        // coded values (vcode.cu): the blob crosses the link instead of the packed values
        const auto* vc = static_cast<const endor_vcode_header*>(op.vcode_host);
        if (vc) {
            if ((st = endor_values_decode_host_check(vc))) return st;
            if (op.path || deq || op.dtype != ENDOR_DTYPE_F16 || vc->nnz != op.nnz)
                return pbad("coded values need an f16 host op whose blob holds exactly nnz values");
            if (vc->blob_bytes > p->max_elems * 2 + 4096) return pbad("coded-values blob larger than the staging slot");
        }
        if (!op.path && ((n && !op.bitmap_host) || (op.nnz && !op.values_host && !vc))) return pbad("null host buffer");
        auto& slot = p->slots[i % p->depth];
        if (vc && !slot.coded) {
            PK(cudaStreamSynchronize(p->copy));
            PK(cudaMalloc(&slot.coded, align256(p->max_elems * 2 + 4096)));
        }
        const size_t bmb = (n + 7) / 8;
        size_t vb = vc ? size_t(vc->blob_bytes) : op.nnz * eb;  // bytes that cross the link / leave storage
        const size_t pb = op.prefix1024_host ? (n + 1023) / 1024 * 8 : 0;
        // copy stream: wait until the slot's previous occupant was decompressed
        NvtxRange h2d_range(op.path ? "endor op: storage -> HBM" : "endor op: H2D compressed");
        PK(cudaStreamWaitEvent(p->copy, slot.free_ev, 0));
        PK(cudaEventRecord(p->h2d_beg[i], p->copy));
        if (op.path) {
            // EndorDirect: storage -> device (the reader's H2D chunks go on the copy stream)
            endor_file_info fi;
            if ((st = endor_file_probe(op.path, &fi))) return st;
            if (fi.rows != op.rows || fi.cols != op.cols || fi.dtype != op.dtype || fi.nnz != op.nnz)
                return pbad("op shape / dtype / nnz disagree with the file header");
            if (!p->reader && (st = endor_reader_create(p->device, 0, ENDOR_IO_AUTO, &p->reader))) return st;
            if ((st = endor_reader_read(p->reader, op.path, &fi, slot.bitmap, slot.values, 0, nullptr, 0, p->copy)))
                return st;
            vb = fi.values_bytes;  // v3 containers: the coded section
        } else {
            PK(cudaMemcpyAsync(slot.bitmap, op.bitmap_host, bmb, cudaMemcpyHostToDevice, p->copy));
            if (vc) PK(cudaMemcpyAsync(slot.coded, vc, vb, cudaMemcpyHostToDevice, p->copy));
            else if (vb) PK(cudaMemcpyAsync(slot.values, op.values_host, vb, cudaMemcpyHostToDevice, p->copy));
        }
        if (pb) PK(cudaMemcpyAsync(slot.prefix, op.prefix1024_host, pb, cudaMemcpyHostToDevice, p->copy));
        const uint64_t* pre = pb ? slot.prefix : nullptr;
        PK(cudaEventRecord(p->h2d_end[i], p->copy));
        // compute stream: decompress into the dense ring (or the caller's buffer), then GEMV
        NvtxRange compute_range("endor op: decompress + GEMV");
        PK(cudaStreamWaitEvent(p->compute, p->h2d_end[i], 0));
        PK(cudaEventRecord(p->dec_beg[i], p->compute));
        if (vc) {  // blob -> packed f16 values in the slot (decode + exception patch)
            if ((st = endor_cuda_values_decode(vc, slot.coded, slot.values, p->compute))) return st;
            launches += vc->n_exc ? 2 : 1;
        }
        endor_tensor_view v{op.rows, op.cols, op.dtype, 0, slot.bitmap, slot.values, op.nnz};
        // y = W x with W never observed by the caller: fused decompress -> GEMV
        // (no dense W in HBM) unless flags bit1 asks for the materialised path
        const bool fused = op.x_dev && op.y_dev && !op.dense_dev && !deq && op.dtype == ENDOR_DTYPE_F16 &&
                           op.cols % 1024 == 0 && !(op.flags & 2);
        if (gemm) {
            // Y = X W^T from the compressed W (fused tcgen05 GEMM; past the
            // two-pass threshold: decompress into the workspace + dense GEMM)
            st = endor_cuda_gemm_compressed(&v, pre, op.x_dev, op.tokens, op.cols, op.y_dev, nullptr, p->ws,
                                            p->ws_bytes, p->compute);
            if (st) return st;
            launches += pre ? 2 : 4;
            PK(cudaEventRecord(p->dec_end[i], p->compute));
            PK(cudaEventRecord(slot.free_ev, p->compute));
        } else if (fused) {
            st = endor_cuda_gemv_compressed(&v, pre, op.x_dev, op.y_dev, nullptr, p->ws, p->ws_bytes, p->compute);
            if (st) return st;
            launches += pre ? 2 : 4;  // (count, flatten,) fused GEMV, row sum
            PK(cudaEventRecord(p->dec_end[i], p->compute));
            PK(cudaEventRecord(slot.free_ev, p->compute));
        } else {
            void* dst = op.dense_dev ? op.dense_dev : p->dense[i & 1];
            st = deq   ? endor_cuda_decompress_dequant(&v, op.quant_scale, dst, p->ws, p->ws_bytes, p->compute)
                 : pre ? endor_cuda_decompress_chunked(&v, 1024, pre, (n + 1023) / 1024, dst, p->ws, p->ws_bytes,
                                                       p->compute)
                       : endor_cuda_decompress(&v, dst, p->ws, p->ws_bytes, p->compute);
            if (st) return st;
            launches += pre ? 1 : 2;
            PK(cudaEventRecord(p->dec_end[i], p->compute));
            PK(cudaEventRecord(slot.free_ev, p->compute));
            if (op.x_dev && op.y_dev) {
                st = endor_cuda_gemv(op.rows, op.cols, dst, op.x_dev, op.y_dev, nullptr, p->compute);
                if (st) return st;
                launches += 1;
            }
        }
        if (op.x_dev && op.y_dev && op.y_host)
            PK(cudaMemcpyAsync(op.y_host, op.y_dev, op.rows * sizeof(float) * (gemm ? op.tokens : 1),
                               cudaMemcpyDeviceToHost, p->compute));
        PK(cudaEventRecord(p->op_end[i], p->compute));
        h2d += bmb + vb + pb;
        dense += n * ob;
    }
    p->last_nops = nops;
    p->last_h2d_bytes = h2d;
    p->last_dense_bytes = dense;
    p->last_launches = launches;
    if (sync) {
        PK(cudaStreamSynchronize(p->compute));
        return endor_cuda_sync_status(p->ws, p->compute);
    }
    return ENDOR_OK;
}

int endor_pipeline_stats_get(endor_pipeline* p, endor_pipeline_stats* out) {
    if (!p || !out) return pbad("null pipeline or output");
    PK(cudaSetDevice(p->device));
    PK(cudaStreamSynchronize(p->compute));
    PK(cudaStreamSynchronize(p->copy));
    endor_pipeline_stats s{};
    const int n = p->last_nops;
    if (n > 0) {
        float ms = 0.f;
        PK(cudaEventElapsedTime(&ms, p->h2d_beg[0], p->op_end[n - 1]));
        s.total_ms = ms;
        float copy_span = 0.f;
        PK(cudaEventElapsedTime(&copy_span, p->h2d_beg[0], p->h2d_end[n - 1]));
        s.exposed_compute_ms = ms - copy_span;
        for (int i = 0; i < n; ++i) {
            PK(cudaEventElapsedTime(&ms, p->h2d_beg[i], p->h2d_end[i]));
            s.h2d_ms += ms;
            PK(cudaEventElapsedTime(&ms, p->dec_beg[i], p->dec_end[i]));
            s.decompress_ms += ms;
            PK(cudaEventElapsedTime(&ms, p->dec_end[i], p->op_end[i]));
            s.gemv_ms += ms;
        }
    }
    s.h2d_bytes = p->last_h2d_bytes;
    s.dense_bytes = p->last_dense_bytes;
    s.kernel_launches = p->last_launches;
    *out = s;
    return ENDOR_OK;
}

}  // extern "C"
