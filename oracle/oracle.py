"""ctypes front-end for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loads ``oracle/liboracle.so`` (the C restatement in ``endor_oracle.c``) and,
when present, ``oracle/_ref/libendor_ref.so`` (the unmodified reference headers
behind ``ref_shim.cpp``).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this module;
the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_u64, _i32, _f64 = C.c_uint64, C.c_int, C.c_double

OK, SIZE, CORRUPTION, BOUNDS, INVALID = 0, 1, 2, 3, 4


def build() -> None:
    """Build liboracle.so (and _ref/ where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(name: str):
    path = os.path.join(HERE, name)
    if not os.path.exists(path):
        if name == "liboracle.so":
            build()
        else:
            return None
    return C.CDLL(path)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load("liboracle.so")
        L = _lib
        L.or_popcount.argtypes = [_u8p, _u64]
        L.or_popcount.restype = _u64
        L.or_rank_range.argtypes = [_u8p, _u64, _u64]
        L.or_rank_range.restype = _u64
        L.or_rank_index.argtypes = [_u8p, _u64, _u64, _u64p]
        L.or_decompress.argtypes = [_u64, _u64, _i32, _u8p, _u8p, _u64, _u8p]
        L.or_check_index.argtypes = [_u64, _u8p, _u64, _u64, _u64p, _u64]
        L.or_decompress_chunk_into.argtypes = [_u64, _u64, _i32, _u8p, _u8p, _u64, _u64, _u64p,
                                               _u64, _u64, _u8p, _u64]
        L.or_decompress_chunked.argtypes = [_u64, _u64, _i32, _u8p, _u8p, _u64, _u64, _u64p,
                                            _u64, _u8p]
        L.or_compress.argtypes = [_u64, _u64, _i32, _u8p, _u8p, _u8p, C.POINTER(_u64),
                                  C.POINTER(_i32)]
        L.or_f16_to_f32.argtypes = [C.c_uint16]
        L.or_f16_to_f32.restype = C.c_float
        L.or_f32_to_f16.argtypes = [C.c_float]
        L.or_f32_to_f16.restype = C.c_uint16
        L.or_synth_weight.argtypes = [_u64, _i32, _u64, _u8p]
        L.or_synth_weight.restype = None
        L.or_magnitude_prune.argtypes = [_u64, _i32, _f64, _u8p, _u8p]
        L.or_nm_prune.argtypes = [_u64, _u64, _i32, _u64, _u64, _u8p, _u8p]
        L.or_random_dense.argtypes = [_u64, _u64, _i32, _u64, _f64, _u8p]
        L.or_random_dense.restype = None
        L.or_mt64_seed.argtypes = [C.c_void_p, _u64]
        L.or_mt64_seed.restype = None
        L.or_mt64_next.argtypes = [C.c_void_p]
        L.or_mt64_next.restype = _u64
        L.or_mt64_coin.argtypes = [C.c_void_p]
        L.or_mt64_coin.restype = _f64
        L.or_acceptance_matrix.argtypes = [C.c_void_p, _u64, _u64, _i32, _f64, _u8p]
        L.or_acceptance_matrix.restype = None
        L.or_dequantize_values.argtypes = [_u8p, _u64, C.c_float, _u16p]
        L.or_dequantize_values.restype = None
        L.or_quantize_values.argtypes = [_u16p, _u64, _u8p]
        L.or_quantize_values.restype = C.c_float
        L.or_make_op_mt.argtypes = [_u64, _u64, _u64, _f64, _i32, _u8p, _u8p]
        L.or_make_op_mt.restype = _u64
        L.or_decompress_parallel.argtypes = [_u64, _i32, _u8p, _u8p, _u64, _u64p, _u8p, _i32]
        L.or_decompress_parallel.restype = _f64
        L.or_gemv_f16.argtypes = [_u64, _u64, _u16p, _u16p, _f32p]
        L.or_gemv_f16.restype = None
    return _lib


def ref():
    """The reference itself (oracle/_ref/libendor_ref.so) or None."""
    global _ref
    if _ref is None:
        _ref = _load(os.path.join("_ref", "libendor_ref.so"))
        if _ref is None:
            return None
        R = _ref
        R.ref_tensor_new.argtypes = [_u64, _u64, _i32, _u8p, _u8p, _u64, C.POINTER(_i32)]
        R.ref_tensor_new.restype = C.c_void_p
        R.ref_tensor_free.argtypes = [C.c_void_p]
        R.ref_tensor_free.restype = None
        R.ref_decompress_timed.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_i32)]
        R.ref_decompress_timed.restype = _f64
        R.ref_decompress_parallel_timed.argtypes = [C.c_void_p, _u64p, _u64, _u64, _i32,
                                                    C.c_void_p, C.POINTER(_i32)]
        R.ref_decompress_parallel_timed.restype = _f64
        R.ref_decompress.argtypes = [_u64, _u64, _i32, _u8p, _u8p, _u64, _u8p]
        R.ref_rank_index.argtypes = [_u8p, _u64, _u64, _u64p]
        R.ref_decompress_chunked.argtypes = [_u64, _u64, _i32, _u8p, _u8p, _u64, _u64, _u64p,
                                             _u64, _u8p]
        R.ref_decompress_chunk_into.argtypes = [_u64, _u64, _i32, _u8p, _u8p, _u64, _u64,
                                                _u64p, _u64, _u64, _u8p, _u64]
        R.ref_compress.argtypes = [_u64, _u64, _i32, _u8p, _u8p, _u8p, C.POINTER(_u64),
                                   C.POINTER(_i32)]
        R.ref_synth_prune.argtypes = [_u64, _u64, _i32, _u64, _f64, _u8p]
        R.ref_nm_prune.argtypes = [_u64, _u64, _i32, _u8p, _u64, _u64, _u8p]
        R.ref_random_dense.argtypes = [_u64, _u64, _i32, _u64, _f64, _u8p]
        R.ref_mt64_draws.argtypes = [_u64, _u64, _u64p,
                                     np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")]
        R.ref_mt64_draws.restype = _u64
        R.ref_encode_endor.argtypes = [_u64, _u64, _i32, _u8p, _u8p, _u64, _i32, _u8p, _u64]
        R.ref_encode_endor.restype = _u64
        R.ref_decode_endor.argtypes = [_u8p, _u64, C.POINTER(_u64), C.POINTER(_u64),
                                       C.POINTER(_i32), C.POINTER(_u64)]
        R.ref_f32_to_f16.argtypes = [C.c_float]
        R.ref_f32_to_f16.restype = C.c_uint16
        R.ref_quantize_values.argtypes = [_u64, _u64, _u8p, _u8p, _u64, _u8p]
        R.ref_quantize_values.restype = C.c_float
        R.ref_decompress_dequant.argtypes = [_u64, _u64, _u8p, _u8p, _u64, C.c_float, _u8p]
        R.ref_extract.argtypes = [_u64, _u64, _i32, _u8p, _u8p, _u64, _u64p, _u64, _i32, _u8p]
    return _ref


# ---- numpy conveniences ---------------------------------------------------

def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a).view(np.uint8).reshape(-1))


def compress(dense: np.ndarray, rows: int, cols: int, eb: int):
    """codec.hpp:97-126 -> (bitmap bytes, values bytes, nnz, negzero)."""
    n = rows * cols
    d = _u8(dense)
    bm = np.zeros((n + 7) // 8, np.uint8)
    vals = np.zeros(max(n * eb, 1), np.uint8)
    nnz, nz = _u64(0), _i32(0)
    st = lib().or_compress(rows, cols, eb, d, bm, vals, C.byref(nnz), C.byref(nz))
    assert st == OK
    return bm, vals[: nnz.value * eb].copy(), nnz.value, bool(nz.value)


def decompress(rows, cols, eb, bitmap, values, nnz):
    n = rows * cols
    out = np.zeros(max(n * eb, 1), np.uint8)
    st = lib().or_decompress(rows, cols, eb, _u8(bitmap) if len(bitmap) else np.zeros(1, np.uint8),
                             _u8(values) if len(values) else np.zeros(1, np.uint8), nnz, out)
    return st, out[: n * eb]


def rank_index(bitmap, n, cs):
    chunks = 0 if (n == 0 or cs == 0) else (n + cs - 1) // cs
    out = np.zeros(max(chunks, 1), np.uint64)
    st = lib().or_rank_index(_u8(bitmap) if len(bitmap) else np.zeros(1, np.uint8), n, cs, out)
    return st, out[:chunks]


def synth_weight(rows, cols, eb, seed):
    out = np.zeros(max(rows * cols * eb, 1), np.uint8)
    lib().or_synth_weight(rows * cols, eb, seed, out)
    return out[: rows * cols * eb]


def magnitude_prune(w, n, eb, sparsity):
    out = np.zeros(max(n * eb, 1), np.uint8)
    st = lib().or_magnitude_prune(n, eb, sparsity, _u8(w), out)
    return st, out[: n * eb]


def random_dense(rows, cols, eb, seed, zero_fraction):
    out = np.zeros(max(rows * cols * eb, 1), np.uint8)
    lib().or_random_dense(rows, cols, eb, seed, zero_fraction, out)
    return out[: rows * cols * eb]


class MT64:
    """std::mt19937_64 (+ libstdc++ uniform_real_distribution<double>(0,1))."""

    def __init__(self, seed: int):
        self._buf = C.create_string_buffer(312 * 8 + 16)
        lib().or_mt64_seed(self._buf, seed)

    def __call__(self) -> int:
        return lib().or_mt64_next(self._buf)

    def coin(self) -> float:
        return lib().or_mt64_coin(self._buf)

    def acceptance_matrix(self, rows, cols, eb, zf):
        out = np.zeros(max(rows * cols * eb, 1), np.uint8)
        lib().or_acceptance_matrix(self._buf, rows, cols, eb, zf, out)
        return out[: rows * cols * eb]


def acceptance_cases(count: int = 1000):
    """Replays acceptance.cpp:99-157's generator: yields
    (iter, rows, cols, eb, zeros, dense_bytes, chunk)."""
    g = MT64(20240521)
    for it in range(count):
        big = it % 50 == 0
        rows = 1 + g() % (160 if big else 48)
        cols = 1 + g() % (160 if big else 48)
        eb = 2 if g() % 2 else 1
        zeros = (g() % 101) / 100.0
        w = g.acceptance_matrix(rows, cols, eb, zeros)
        chunk = 64 << (g() % 7)
        rsel = [r for r in range(rows) if g.coin() < 0.5]
        csel = [c for c in range(cols) if g.coin() < 0.5]
        yield it, rows, cols, eb, zeros, w, chunk, rsel, csel


def quantize_values(vals_u8: np.ndarray, nnz: int):
    """codec.hpp:306-331 -> (i8 bytes, scale)."""
    v16 = np.ascontiguousarray(vals_u8).view(np.uint16) if nnz else np.zeros(1, np.uint16)
    q = np.zeros(max(nnz, 1), np.uint8)
    scale = lib().or_quantize_values(v16, nnz, q)
    return q[:nnz], scale


def decompress_dequant(rows, cols, bitmap, q, nnz, scale):
    """decompress(dequantize_values(t)) on the CPU oracle -> f16 dense bytes."""
    h = np.zeros(max(nnz, 1), np.uint16)
    lib().or_dequantize_values(np.ascontiguousarray(q) if nnz else np.zeros(1, np.uint8), nnz, scale, h)
    return decompress(rows, cols, 2, bitmap, h[:nnz].view(np.uint8), nnz)


def gemv_f16(w_u16: np.ndarray, x_u16: np.ndarray, rows: int, cols: int) -> np.ndarray:
    y = np.zeros(max(rows, 1), np.float32)
    lib().or_gemv_f16(rows, cols, np.ascontiguousarray(w_u16.reshape(-1)),
                      np.ascontiguousarray(x_u16.reshape(-1)), y)
    return y[:rows]
