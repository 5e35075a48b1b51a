/* The C calls INTEGRATION.md §3 shows, with their variables declared:
 * type-checked against include/endor_cuda.h by tests/test_capi.py
 * (gcc -fsyntax-only; nothing here runs). */
#include <stddef.h>
#include <stdint.h>

#include "endor_cuda.h"

int integration_example(uint64_t rows, uint64_t cols, uint64_t nnz, const void* d_bitmap, const void* d_values,
                        void* d_dense, void* ws, void* stream, const void* h_bitmap, const void* h_values,
                        const void* d_x, float* d_y, float* h_y, const char* path, const uint64_t* d_rows,
                        const uint64_t* d_cols, uint64_t nsel, void* d_out, const void* d_vals_f16, void* d_q,
                        void* d_vals_out, const endor_tensor_view* views, const uint64_t* const* idx1024,
                        const void* const* xs, float* const* ys, const void* const* dense_ws,
                        const uint64_t* op_rows, const uint64_t* op_cols) {
    endor_tensor_view t = {rows, cols, ENDOR_DTYPE_F16, 0, d_bitmap, d_values, nnz};
    size_t ws_bytes = endor_cuda_workspace_bytes(rows, cols);
    int st = endor_cuda_workspace_init(ws, ws_bytes, stream);
    st |= endor_cuda_decompress(&t, d_dense, ws, ws_bytes, stream);
    st |= endor_cuda_sync_status(ws, stream);
    void* outs[6] = {d_dense, d_dense, d_dense, d_dense, d_dense, d_dense};
    st |= endor_cuda_decompress_batch(views, outs, 6, ws, endor_cuda_workspace_bytes_batch(views, 6), stream);

    endor_pipeline* p;
    st |= endor_pipeline_create(0, rows * cols, 2, &p);
    endor_pipeline_op ops[1] = {{rows, cols, ENDOR_DTYPE_F16, 0, h_bitmap, h_values, nnz, d_x, d_y, NULL, h_y}};
    st |= endor_pipeline_run(p, ops, 1, /*sync=*/1);
    endor_pipeline_stats s;
    st |= endor_pipeline_stats_get(p, &s);

    st |= endor_cuda_gemv_compressed_batch(views, idx1024, xs, ys, NULL, 6, ws,
                                           endor_cuda_workspace_bytes_batch(views, 6), stream);
    st |= endor_cuda_gemv_batch(op_rows, op_cols, dense_ws, xs, ys, NULL, 6, stream);

    const uint64_t tokens = 16, x_ld = cols;
    const size_t gws = endor_cuda_gemm_workspace_bytes(rows, cols, tokens);
    st |= endor_cuda_gemm_compressed(&t, NULL, d_x, tokens, x_ld, d_y, NULL, ws, gws, stream);
    st |= endor_cuda_gemm(rows, cols, d_dense, d_x, tokens, x_ld, d_y, NULL, ws, gws, stream);
    endor_pipeline_op gop = {0};
    gop.tokens = tokens;
    gop.prefix1024_host = NULL;
    (void)gop;
    size_t v2 = endor_file_encode_v2(rows, cols, ENDOR_DTYPE_F16, 0, 0.f, h_bitmap, h_values, nnz, NULL, 0);
    (void)v2;

    st |= endor_cuda_extract_rows(&t, d_rows, nsel, d_out, ws, ws_bytes, stream);
    st |= endor_cuda_extract_cols(&t, d_cols, nsel, d_out, ws, ws_bytes, stream);
    float scale;
    st |= endor_cuda_quantize_values(d_vals_f16, nnz, d_q, &scale, ws, ws_bytes, stream);
    endor_tensor_view t_i8 = {rows, cols, ENDOR_DTYPE_I8, 0, d_bitmap, d_q, nnz};
    st |= endor_cuda_decompress_dequant(&t_i8, scale, d_dense, ws, ws_bytes, stream);
    st |= endor_cuda_dequantize_values(d_q, nnz, scale, d_vals_out, stream);

    endor_file_info f;
    if (endor_file_probe(path, &f)) st |= endor_cuda_last_format_kind();
    endor_reader* r;
    st |= endor_reader_create(0, 0, ENDOR_IO_AUTO, &r);
    st |= endor_reader_read(r, path, &f, d_dense, d_vals_out, /*verify=*/1, ws, ws_bytes, stream);
    endor_pipeline_op op = {0};
    op.rows = f.rows;
    op.cols = f.cols;
    op.dtype = f.dtype;
    op.nnz = f.nnz;
    op.x_dev = d_x;
    op.y_dev = d_y;
    op.path = path;
    size_t nb = 0;
    st |= endor_values_encode(h_values, nnz, 7, NULL, 0, &nb);
    void* blob = endor_host_alloc(nb);
    st |= endor_values_encode(h_values, nnz, 7, blob, nb, &nb);
    endor_pipeline_op cop = ops[0];
    cop.values_host = NULL;
    cop.vcode_host = blob;
    st |= endor_cuda_values_decode(blob, d_dense, d_vals_out, stream);
    st |= endor_pipeline_run(p, &cop, 1, 1);
    endor_host_free(blob);
    st |= endor_reader_destroy(r);
    st |= endor_pipeline_destroy(p);
    return st + (int)op.rows;
}
