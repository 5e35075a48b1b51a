"""ctypes binding of the C ABI in include/endor_cuda.h (libendor_cuda.so).

There is no fallback: if the shared library is missing or cannot be loaded,
every entry point raises.  The library is built in-tree by
``paper_2406_11674_b200/build.py`` (``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
# ENDOR_LIB: load a differently-built copy (development variants, tools/build_variant.sh)
LIB_PATH = os.environ.get("ENDOR_LIB") or os.path.join(PKG, "libendor_cuda.so")

_u64, _i32, _vp, _sz, _f64 = C.c_uint64, C.c_int32, C.c_void_p, C.c_size_t, C.c_double


class TensorView(C.Structure):
    """endor_tensor_view (include/endor_cuda.h)."""
    _fields_ = [("rows", _u64), ("cols", _u64), ("dtype", _i32), ("reserved", _i32),
                ("bitmap", _vp), ("values", _vp), ("nnz", _u64)]


class PipelineOp(C.Structure):
    """endor_pipeline_op."""
    _fields_ = [("rows", _u64), ("cols", _u64), ("dtype", _i32), ("flags", _i32),
                ("bitmap_host", _vp), ("values_host", _vp), ("nnz", _u64),
                ("x_dev", _vp), ("y_dev", _vp), ("dense_dev", _vp), ("y_host", _vp),
                ("quant_scale", C.c_float), ("reserved2", _i32), ("path", C.c_char_p),
                ("tokens", _u64), ("prefix1024_host", _vp), ("vcode_host", _vp)]


class PipelineStats(C.Structure):
    """endor_pipeline_stats."""
    _fields_ = [("total_ms", _f64), ("h2d_ms", _f64), ("decompress_ms", _f64), ("gemv_ms", _f64),
                ("exposed_compute_ms", _f64), ("h2d_bytes", _u64), ("dense_bytes", _u64),
                ("kernel_launches", _u64)]


class FileInfo(C.Structure):
    """endor_file_info."""
    _fields_ = [("rows", _u64), ("cols", _u64), ("nnz", _u64), ("dtype", _i32), ("flags", _i32),
                ("quant_scale", C.c_float), ("crc", C.c_uint32), ("header_crc", C.c_uint32),
                ("gap_bytes", C.c_uint32), ("header_bytes", _u64), ("bitmap_offset", _u64),
                ("bitmap_bytes", _u64), ("values_offset", _u64), ("values_bytes", _u64), ("file_bytes", _u64),
                ("values_out_bytes", _u64)]


# name -> (restype, argtypes): every symbol include/endor_cuda.h declares
SIGNATURES = {
    "endor_cuda_abi_version": (C.c_int, []),
    "endor_cuda_last_error_string": (C.c_char_p, []),
    "endor_cuda_status_name": (C.c_char_p, [C.c_int]),
    "endor_cuda_tile_elems": (_u64, []),
    "endor_cuda_workspace_bytes": (_sz, [_u64, _u64]),
    "endor_cuda_workspace_init": (C.c_int, [_vp, _sz, _vp]),
    "endor_cuda_sync_status": (C.c_int, [_vp, _vp]),
    "endor_cuda_decompress": (C.c_int, [C.POINTER(TensorView), _vp, _vp, _sz, _vp]),
    "endor_cuda_workspace_bytes_batch": (_sz, [C.POINTER(TensorView), C.c_int]),
    "endor_cuda_decompress_batch": (C.c_int, [C.POINTER(TensorView), C.POINTER(_vp), C.c_int, _vp, _sz,
                                              _vp]),
    "endor_cuda_decompress_batch_phase": (C.c_int, [C.POINTER(TensorView), C.POINTER(_vp), C.c_int,
                                                    C.c_int, _vp, _sz, _vp]),
    "endor_cuda_decompress_chunked_batch": (C.c_int, [C.POINTER(TensorView), C.POINTER(_vp), _u64,
                                                      C.POINTER(_vp), C.c_int, _vp, _sz, _vp]),
    "endor_cuda_decompress_dequant": (C.c_int, [C.POINTER(TensorView), C.c_float, _vp, _vp, _sz, _vp]),
    "endor_cuda_gemm_workspace_bytes": (_sz, [_u64, _u64, _u64]),
    "endor_cuda_gemm": (C.c_int, [_u64, _u64, _vp, _vp, _u64, _u64, _vp, _vp, _vp, _sz, _vp]),
    "endor_cuda_gemm_compressed": (C.c_int, [C.POINTER(TensorView), _vp, _vp, _u64, _u64, _vp, _vp, _vp, _sz,
                                             _vp]),
    "endor_cuda_gemv_compressed": (C.c_int, [C.POINTER(TensorView), _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "endor_cuda_gemv_compressed_batch": (C.c_int, [C.POINTER(TensorView), C.POINTER(_vp), C.POINTER(_vp),
                                                   C.POINTER(_vp), C.POINTER(_vp), C.c_int, _vp, _sz, _vp]),
    "endor_cuda_extract_rows": (C.c_int, [C.POINTER(TensorView), _vp, _u64, _vp, _vp, _sz, _vp]),
    "endor_cuda_extract_cols": (C.c_int, [C.POINTER(TensorView), _vp, _u64, _vp, _vp, _sz, _vp]),
    "endor_cuda_decompress_phase": (C.c_int, [C.POINTER(TensorView), _vp, C.c_int, _vp, _sz, _vp]),
    "endor_cuda_rank_index": (C.c_int, [_vp, _u64, _u64, _vp, _vp, _vp, _sz, _vp]),
    "endor_cuda_popcount": (C.c_int, [_vp, _u64, _vp, _vp, _sz, _vp]),
    "endor_cuda_decompress_chunked": (C.c_int, [C.POINTER(TensorView), _u64, _vp, _u64, _vp, _vp,
                                                _sz, _vp]),
    "endor_cuda_decompress_chunk_into": (C.c_int, [C.POINTER(TensorView), _u64, _vp, _u64, _u64,
                                                   _vp, _u64, _vp, _sz, _vp]),
    "endor_cuda_decompress_host": (C.c_int, [_u64, _u64, _i32, _vp, _vp, _u64, _vp]),
    "endor_cuda_rank_index_host": (C.c_int, [_vp, _u64, _u64, _vp]),
    "endor_cuda_decompress_chunked_host": (C.c_int, [_u64, _u64, _i32, _vp, _vp, _u64, _u64, _vp,
                                                     _u64, _vp]),
    "endor_cuda_decompress_chunk_into_host": (C.c_int, [_u64, _u64, _i32, _vp, _vp, _u64, _u64, _vp,
                                                        _u64, _u64, _vp, _u64]),
    "endor_cuda_compress_host": (C.c_int, [_u64, _u64, _i32, _vp, _vp, _vp, C.POINTER(_u64),
                                           C.POINTER(_i32)]),
    "endor_cuda_compress": (C.c_int, [_u64, _u64, _i32, _vp, _vp, _vp, C.POINTER(_u64),
                                      C.POINTER(_i32), _vp, _sz, _vp]),
    "endor_cuda_quantize_values": (C.c_int, [_vp, _u64, _vp, C.POINTER(C.c_float), _vp, _sz, _vp]),
    "endor_cuda_dequantize_values": (C.c_int, [_vp, _u64, C.c_float, _vp, _vp]),
    "endor_cuda_extract_rows_host": (C.c_int, [_u64, _u64, _i32, _vp, _vp, _u64, _vp, _u64, _vp]),
    "endor_cuda_extract_cols_host": (C.c_int, [_u64, _u64, _i32, _vp, _vp, _u64, _vp, _u64, _vp]),
    "endor_cuda_quantize_values_host": (C.c_int, [_vp, _u64, _vp, C.POINTER(C.c_float)]),
    "endor_cuda_dequantize_values_host": (C.c_int, [_vp, _u64, C.c_float, _vp]),
    "endor_cuda_synth_weight": (C.c_int, [_u64, _u64, _i32, _u64, _u64, _u64, _vp, _vp]),
    "endor_cuda_magnitude_prune": (C.c_int, [_u64, _i32, _f64, _vp, _vp, _sz, _vp]),
    "endor_cuda_gemv": (C.c_int, [_u64, _u64, _vp, _vp, _vp, _vp, _vp]),
    "endor_cuda_gemv_batch": (C.c_int, [C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_vp), C.POINTER(_vp),
                                        C.POINTER(_vp), C.POINTER(_vp), C.c_int, _vp]),
    "endor_pipeline_create": (C.c_int, [C.c_int, _u64, C.c_int, C.POINTER(_vp)]),
    "endor_pipeline_destroy": (C.c_int, [_vp]),
    "endor_pipeline_run": (C.c_int, [_vp, C.POINTER(PipelineOp), C.c_int, C.c_int]),
    "endor_pipeline_stats_get": (C.c_int, [_vp, C.POINTER(PipelineStats)]),
    "endor_pipeline_stream": (_vp, [_vp]),
    "endor_cuda_last_format_kind": (C.c_int, []),
    "endor_file_probe": (C.c_int, [C.c_char_p, C.POINTER(FileInfo)]),
    "endor_file_encode": (_sz, [_u64, _u64, _i32, _i32, C.c_float, _vp, _vp, _u64, _vp, _sz]),
    "endor_file_encode_v2": (_sz, [_u64, _u64, _i32, _i32, C.c_float, _vp, _vp, _u64, _vp, _sz]),
    "endor_file_encode_v3": (_sz, [_u64, _u64, _i32, _vp, _vp, _u64, _vp, _sz]),
    "endor_reader_create": (C.c_int, [C.c_int, _sz, C.c_int, C.POINTER(_vp)]),
    "endor_reader_destroy": (C.c_int, [_vp]),
    "endor_reader_mode": (C.c_int, [_vp]),
    "endor_reader_read": (C.c_int, [_vp, C.c_char_p, C.POINTER(FileInfo), _vp, _vp, C.c_int, _vp, _sz, _vp]),
    "endor_reader_stats": (C.c_int, [_vp, C.POINTER(_f64), C.POINTER(_u64)]),
    "endor_values_encode": (C.c_int, [_vp, _u64, C.c_int, _vp, _sz, C.POINTER(_sz)]),
    "endor_values_decode_host_check": (C.c_int, [_vp]),
    "endor_cuda_values_decode": (C.c_int, [_vp, _vp, _vp, _vp]),
    "endor_host_alloc": (_vp, [_sz]),
    "endor_host_free": (None, [_vp]),
}

_lock = threading.Lock()
_lib = None


def lib():
    """Load libendor_cuda.so (raises if absent -- no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback for the Endor CUDA path)")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib
