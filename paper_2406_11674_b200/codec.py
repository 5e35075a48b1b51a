"""Host-side mirror of the reference's codec API over the CUDA C ABI.

Same names, argument meaning and error types as the reference's
``proj/include/endor/`` headers, so parity tests read like the reference's
own tests.  Data lives in device memory (torch uint8 tensors are used purely
as allocations + stream plumbing); every compute call goes through
``libendor_cuda.so`` -- there is no CPU path.

Reference anchors:
  EndorTensor              codec.hpp:24-66
  compression_ratio etc.   codec.hpp:75-88
  compress                 codec.hpp:97-126       -> endor_cuda_compress
  decompress               codec.hpp:157-166      -> endor_cuda_decompress
  decompress_chunk_into    codec.hpp:191-201      -> endor_cuda_decompress_chunk_into
  decompress_chunked       codec.hpp:205-216      -> endor_cuda_decompress_chunked
  Bitmap / RankIndex       bitmap.hpp:18-132      -> endor_cuda_popcount / _rank_index
  DenseMatrix / Dtype      dense_matrix.hpp:18-99
  synth_weight / magnitude_prune  weight_gen.hpp:40-113
  error classes            error.hpp:9-63
"""
from __future__ import annotations

import ctypes as C
import threading
import enum
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import torch

from . import _lib
from ._lib import TensorView


# ---- errors (error.hpp:9-63) -----------------------------------------------

class Error(RuntimeError):
    """endor::Error."""


class SizeError(Error):
    """endor::SizeError."""


class CorruptionError(Error):
    """endor::CorruptionError."""


class BoundsError(Error):
    """endor::BoundsError."""


class ConfigError(Error):
    """endor::ConfigError."""


class CudaError(Error):
    """A CUDA runtime failure (no reference analogue)."""


class InvalidArgument(ValueError):
    """std::invalid_argument."""


class FormatError(Error):
    """endor::FormatError (error.hpp:42-60) with its Kind."""

    class Kind(enum.IntEnum):
        Truncated = 0
        BadMagic = 1
        BadVersion = 2
        BadCrc = 3
        CountMismatch = 4
        Malformed = 5

    def __init__(self, msg: str, kind: "FormatError.Kind"):
        super().__init__(msg)
        self.kind = kind


_STATUS = {1: SizeError, 2: CorruptionError, 3: BoundsError, 4: InvalidArgument, 5: CudaError,
           6: ConfigError, 8: Error}


def check(status: int) -> None:
    if status != 0:
        L = _lib.lib()
        msg = L.endor_cuda_last_error_string().decode(errors="replace")
        if status == 7:
            raise FormatError(msg, FormatError.Kind(L.endor_cuda_last_format_kind()))
        raise _STATUS.get(status, Error)(msg)


# ---- dtype (dense_matrix.hpp:18-23) -----------------------------------------

class Dtype(enum.IntEnum):
    F16 = 0
    I8 = 1


def elem_bytes(dtype: Dtype) -> int:
    return 2 if dtype == Dtype.F16 else 1


def checked_element_count(rows: int, cols: int) -> int:
    """dense_matrix.hpp:28-33."""
    if rows < 0 or cols < 0 or (rows != 0 and cols > (2 ** 64 - 1) // rows):
        raise SizeError("matrix dimensions overflow the addressable element count")
    return rows * cols


# ---- size arithmetic (codec.hpp:75-88) --------------------------------------

def compression_ratio(dtype: Dtype, sparsity: float) -> float:
    if not (0.0 <= sparsity <= 1.0):
        raise InvalidArgument("sparsity must be in [0, 1]")
    return (1.0 - sparsity) + 1.0 / (8.0 * elem_bytes(dtype))


def endor_values_bytes(dtype: Dtype, nnz: int) -> int:
    return nnz * elem_bytes(dtype)


def endor_bitmap_bytes(rows: int, cols: int) -> int:
    return (checked_element_count(rows, cols) + 7) // 8


# ---- device plumbing ----------------------------------------------------------

def _dev(device=None) -> torch.device:
    d = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if d.type != "cuda":
        raise InvalidArgument("the Endor path runs on CUDA devices only")
    if d.index is None:
        d = torch.device("cuda", torch.cuda.current_device())
    return d


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None or t.numel() == 0 else t.data_ptr()


def _alloc(nbytes: int, device: torch.device, pad: int = 16) -> torch.Tensor:
    """uint8 device buffer of nbytes (+pad so 16-byte vector loads stay inside)."""
    return torch.empty(nbytes + pad, dtype=torch.uint8, device=device)[:nbytes]


_WS: Dict[Tuple[int, int, int], torch.Tensor] = {}


def workspace(n: int, device: torch.device, min_bytes: int = 0) -> torch.Tensor:
    """Zero-initialised workspace for tensors of up to n elements (and at
    least min_bytes), one per (device, stream, host thread), grown on demand --
    the library leaves it zeroed after every call.  Per thread because host
    threads sharing a stream would interleave their launch sequences (the
    reference allows concurrent per-chunk calls, codec.hpp:188-190)."""
    key = (device.index, _stream_ptr(device), threading.get_ident())
    need = max(_lib.lib().endor_cuda_workspace_bytes(max(n, 1), 1), min_bytes)
    ws = _WS.get(key)
    if ws is None or ws.numel() < need:
        ws = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def sync_status(ws: torch.Tensor, device: torch.device) -> None:
    check(_lib.lib().endor_cuda_sync_status(ws.data_ptr(), _stream_ptr(device)))


# ---- data model ------------------------------------------------------------------

@dataclass
class DenseMatrix:
    """Row-major raw-byte matrix on the device (dense_matrix.hpp:38-99)."""
    rows: int
    cols: int
    dtype: Dtype
    data: torch.Tensor  # uint8, rows*cols*elem_bytes

    @classmethod
    def empty(cls, rows, cols, dtype=Dtype.F16, device=None) -> "DenseMatrix":
        n = checked_element_count(rows, cols)
        return cls(rows, cols, Dtype(dtype), _alloc(n * elem_bytes(dtype), _dev(device)))

    @classmethod
    def from_host(cls, rows, cols, dtype, data, device=None) -> "DenseMatrix":
        n = checked_element_count(rows, cols)
        if isinstance(data, torch.Tensor):
            buf = data.reshape(-1).view(torch.uint8)
        else:
            raw = bytearray(bytes(data))
            buf = torch.frombuffer(raw, dtype=torch.uint8) if raw else torch.zeros(0, dtype=torch.uint8)
        if buf.numel() != n * elem_bytes(dtype):
            raise SizeError("dense data length does not match rows*cols*elem_bytes")
        out = cls.empty(rows, cols, dtype, device)
        out.data.copy_(buf)
        return out

    @property
    def element_count(self) -> int:
        return self.rows * self.cols

    def elem_size(self) -> int:
        return elem_bytes(self.dtype)

    def size_bytes(self) -> int:
        return self.data.numel()

    def bytes(self) -> bytes:
        return self.data.cpu().numpy().tobytes()

    def __eq__(self, o) -> bool:  # bytewise, dense_matrix.hpp:90-92
        return (isinstance(o, DenseMatrix) and self.rows == o.rows and self.cols == o.cols and
                self.dtype == o.dtype and torch.equal(self.data.cpu(), o.data.cpu()))


class Bitmap:
    """Position bitmap on the device: ceil(size/8) LSB-first bytes
    (bitmap.hpp:14-17)."""

    def __init__(self, bit_count: int, data: Optional[torch.Tensor] = None, device=None):
        self._n = int(bit_count)
        nbytes = (self._n + 7) // 8
        if data is None:
            data = torch.zeros(nbytes + 16, dtype=torch.uint8, device=_dev(device))[:nbytes]
        self.data = data

    def size(self) -> int:
        return self._n

    def byte_size(self) -> int:
        return (self._n + 7) // 8

    @classmethod
    def from_bytes(cls, data, bit_count: int, device=None) -> "Bitmap":
        """bitmap.hpp:72-86: exact length and zero padding bits required."""
        raw = bytes(data) if not isinstance(data, torch.Tensor) else data.cpu().numpy().tobytes()
        if len(raw) != (bit_count + 7) // 8:
            raise CorruptionError("bitmap byte length does not match bit count")
        used = bit_count & 7
        if used and raw and (raw[-1] >> used):
            raise CorruptionError("bitmap has nonzero padding bits")
        b = cls(bit_count, device=device)
        if raw:
            b.data.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
        return b

    def to_bytes(self) -> bytes:
        return self.data.cpu().numpy().tobytes()

    def count(self) -> int:
        """bitmap.hpp:34-38 (device popcount)."""
        dev = self.data.device
        out = torch.zeros(1, dtype=torch.int64, device=dev)
        ws = workspace(self._n, dev)
        check(_lib.lib().endor_cuda_popcount(_ptr(self.data), self._n, out.data_ptr(), ws.data_ptr(),
                                             ws.numel(), _stream_ptr(dev)))
        sync_status(ws, dev)
        return int(out.item())

    def __eq__(self, o) -> bool:
        return isinstance(o, Bitmap) and self._n == o._n and torch.equal(self.data.cpu(), o.data.cpu())


@dataclass
class RankIndex:
    """Exclusive per-chunk popcount prefix (bitmap.hpp:101-114), device u64."""
    chunk_size: int
    prefix: torch.Tensor  # int64 (bit-identical to u64 for these ranges)

    def chunk_count(self) -> int:
        return self.prefix.numel()


class EndorTensor:
    """Compressed tensor (codec.hpp:24-66): bitmap + packed row-major values."""

    def __init__(self, rows: int, cols: int, dtype: Dtype, bitmap: Bitmap, values: torch.Tensor,
                 quant_scale: Optional[float] = None, negative_zero_collapsed: bool = False,
                 validate: bool = True, nnz: Optional[int] = None):
        self.rows, self.cols, self.dtype = int(rows), int(cols), Dtype(dtype)
        self.bitmap, self.values = bitmap, values.reshape(-1).view(torch.uint8)
        self.quant_scale, self._negzero = quant_scale, bool(negative_zero_collapsed)
        eb = elem_bytes(self.dtype)
        if validate:  # codec.hpp:34-39
            if bitmap.size() != checked_element_count(rows, cols):
                raise CorruptionError("bitmap length does not match rows*cols")
            if self.values.numel() != bitmap.count() * eb:
                raise CorruptionError("values length does not match bitmap popcount")
        self._nnz = self.values.numel() // eb if nnz is None else int(nnz)

    def element_count(self) -> int:
        return self.rows * self.cols

    def nnz(self) -> int:
        return self._nnz

    def negative_zero_collapsed(self) -> bool:
        return self._negzero

    def values_bytes(self) -> int:
        return self.values.numel()

    def bitmap_bytes(self) -> int:
        return self.bitmap.byte_size()

    def compressed_bytes(self) -> int:
        return self.values_bytes() + self.bitmap_bytes()

    def dense_bytes(self) -> int:
        return self.element_count() * elem_bytes(self.dtype)

    def view(self) -> TensorView:
        return TensorView(self.rows, self.cols, int(self.dtype), 0, _ptr(self.bitmap.data),
                          _ptr(self.values), self._nnz)

    @property
    def device(self) -> torch.device:
        return self.bitmap.data.device


# ---- codec ------------------------------------------------------------------------

def compress(w: DenseMatrix) -> EndorTensor:
    """codec.hpp:97-126 on the device."""
    dev = w.data.device
    n = checked_element_count(w.rows, w.cols)
    eb = elem_bytes(w.dtype)
    bm = Bitmap(n, device=dev)
    vals = _alloc(n * eb, dev)
    ws = workspace(n, dev)
    nnz, negz = C.c_uint64(0), C.c_int32(0)
    check(_lib.lib().endor_cuda_compress(w.rows, w.cols, int(w.dtype), _ptr(w.data), _ptr(bm.data),
                                         _ptr(vals), C.byref(nnz), C.byref(negz), ws.data_ptr(),
                                         ws.numel(), _stream_ptr(dev)))
    values = vals[: nnz.value * eb]
    return EndorTensor(w.rows, w.cols, w.dtype, bm, values, None, bool(negz.value), validate=False,
                       nnz=nnz.value)


def decompress(t: EndorTensor, out: Optional[DenseMatrix] = None, sync: bool = True) -> DenseMatrix:
    """codec.hpp:157-166 on the device.  With sync=False the call is
    asynchronous on the current stream and device-detected corruption is only
    reported by a later sync_status()."""
    dev = t.device
    if out is None:
        out = DenseMatrix.empty(t.rows, t.cols, t.dtype, dev)
    ws = workspace(t.element_count(), dev)
    v = t.view()
    check(_lib.lib().endor_cuda_decompress(C.byref(v), _ptr(out.data), ws.data_ptr(), ws.numel(),
                                           _stream_ptr(dev)))
    if sync:
        sync_status(ws, dev)
    return out


def decompress_dequant(t: EndorTensor, out: Optional[DenseMatrix] = None) -> DenseMatrix:
    """decompress(dequantize_values(t)) fused on the device (codec.hpp:334-349
    then :157): an I8 tensor with quant_scale -> f16 dense, bit-exact."""
    if t.dtype != Dtype.I8 or t.quant_scale is None:  # codec.hpp:335-337
        raise InvalidArgument("dequantize_values requires a quantized i8 tensor")
    dev = t.device
    if out is None:
        out = DenseMatrix.empty(t.rows, t.cols, Dtype.F16, dev)
    ws = workspace(t.element_count(), dev)
    v = t.view()
    check(_lib.lib().endor_cuda_decompress_dequant(C.byref(v), float(t.quant_scale), _ptr(out.data),
                                                   ws.data_ptr(), ws.numel(), _stream_ptr(dev)))
    sync_status(ws, dev)
    return out


def gemv_compressed(t: EndorTensor, x: torch.Tensor, index: Optional[RankIndex] = None,
                    out_f32: Optional[torch.Tensor] = None) -> torch.Tensor:
    """y = W x straight from the compressed W (fused decompress -> GEMV, the
    dense W is never written).  f16 W with cols % 1024 == 0; fp32 result."""
    dev = t.device
    if t.dtype != Dtype.F16 or x.dtype != torch.float16 or x.numel() != t.cols:
        raise InvalidArgument("gemv_compressed needs an f16 W [rows, cols] and f16 x [cols]")
    y = out_f32 if out_f32 is not None else torch.empty(t.rows, dtype=torch.float32, device=dev)
    ws = workspace(t.element_count(), dev)
    pre = None
    if index is not None:
        if index.chunk_size != 1024:
            raise InvalidArgument("gemv_compressed takes a RankIndex at chunk size 1024")
        pre = index.prefix.to(device=dev, dtype=torch.int64).contiguous()
    xc = x.contiguous()
    v = t.view()
    check(_lib.lib().endor_cuda_gemv_compressed(C.byref(v), _ptr(pre), _ptr(xc), _ptr(y), None, ws.data_ptr(),
                                                ws.numel(), _stream_ptr(dev)))
    sync_status(ws, dev)
    return y


def gemm_compressed(t: EndorTensor, x: torch.Tensor, index: Optional[RankIndex] = None,
                    out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """Y = X W^T straight from the compressed W (fused decompress -> tcgen05
    GEMM; the dense W is never written): x f16 [tokens, cols] -> Y [tokens,
    rows] in fp32 (or f16) with fp32 accumulation."""
    dev = t.device
    if t.dtype != Dtype.F16 or x.dtype != torch.float16 or x.dim() != 2 or x.shape[1] != t.cols:
        raise InvalidArgument("gemm_compressed needs an f16 W [rows, cols] and f16 X [tokens, cols]")
    tokens = x.shape[0]
    ld = (t.cols + 7) // 8 * 8
    if x.stride(1) == 1 and x.stride(0) == ld and x.data_ptr() % 16 == 0:
        xc = x
    else:  # TMA rows must be 16-byte strided: pad each row to a multiple of 8 elements
        xc = torch.zeros((tokens, ld), dtype=torch.float16, device=dev)
        xc[:, :t.cols] = x
    y = torch.empty((tokens, t.rows), dtype=out_dtype, device=dev)
    if out_dtype not in (torch.float32, torch.float16):
        raise InvalidArgument("gemm_compressed: out_dtype must be float32 or float16")
    L = _lib.lib()
    ws = workspace(t.element_count(), dev, L.endor_cuda_gemm_workspace_bytes(t.rows, t.cols, tokens))
    pre = None
    if index is not None:
        if index.chunk_size != 1024:
            raise InvalidArgument("gemm_compressed takes a RankIndex at chunk size 1024")
        pre = index.prefix.to(device=dev, dtype=torch.int64).contiguous()
    v = t.view()
    y32, y16 = (y, None) if out_dtype == torch.float32 else (None, y)
    check(L.endor_cuda_gemm_compressed(C.byref(v), _ptr(pre), _ptr(xc), tokens, ld, _ptr(y32), _ptr(y16),
                                       ws.data_ptr(), ws.numel(), _stream_ptr(dev)))
    sync_status(ws, dev)
    return y


def gemm(w: DenseMatrix, x: torch.Tensor, out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """Y = X W^T for a dense f16 W [rows, cols] (cols % 8 == 0) on the tcgen05
    tensor cores (no cuBLAS): x f16 [tokens, cols] -> Y [tokens, rows]."""
    dev = w.data.device
    rows, cols = w.rows, w.cols
    if w.dtype != Dtype.F16 or x.dtype != torch.float16 or x.dim() != 2 or x.shape[1] != cols:
        raise InvalidArgument("gemm needs an f16 W [rows, cols] and f16 X [tokens, cols]")
    if out_dtype not in (torch.float32, torch.float16):
        raise InvalidArgument("gemm: out_dtype must be float32 or float16")
    tokens = x.shape[0]
    xc = x.contiguous()
    y = torch.empty((tokens, rows), dtype=out_dtype, device=dev)
    L = _lib.lib()
    ws = workspace(1, dev, L.endor_cuda_gemm_workspace_bytes(rows, cols, tokens))
    y32, y16 = (y, None) if out_dtype == torch.float32 else (None, y)
    check(L.endor_cuda_gemm(rows, cols, _ptr(w.data), _ptr(xc), tokens, cols, _ptr(y32), _ptr(y16), ws.data_ptr(),
                            ws.numel(), _stream_ptr(dev)))
    sync_status(ws, dev)
    return y


def gemv_compressed_batch(tensors: Sequence[EndorTensor], xs: Sequence[torch.Tensor],
                          indices: Optional[Sequence[Optional[RankIndex]]] = None) -> List[torch.Tensor]:
    """y_i = W_i x_i for a batch (e.g. one decoder layer's ops) in one fused
    decompress -> GEMV launch; indices: optional 1024-chunk RankIndex per
    tensor (None entries are counted on the device)."""
    if len(tensors) != len(xs) or (indices is not None and len(indices) != len(tensors)):
        raise InvalidArgument("one x (and optional index) per tensor")
    if not tensors:
        return []
    dev = tensors[0].device
    ys, keep = [], []
    for t, x in zip(tensors, xs):
        if t.dtype != Dtype.F16 or x.dtype != torch.float16 or x.numel() != t.cols:
            raise InvalidArgument("gemv_compressed_batch needs f16 W [rows, cols] and f16 x [cols]")
        ys.append(torch.empty(t.rows, dtype=torch.float32, device=dev))
        keep.append(x.contiguous())
    pres = []
    for i in range(len(tensors)):
        ix = indices[i] if indices is not None else None
        if ix is not None and ix.chunk_size != 1024:
            raise InvalidArgument("gemv_compressed_batch takes RankIndex entries at chunk size 1024")
        pres.append(None if ix is None else ix.prefix.to(device=dev, dtype=torch.int64).contiguous())
    n = len(tensors)
    views = (_lib.TensorView * n)(*[t.view() for t in tensors])
    P = C.c_void_p
    pre_arr = (P * n)(*[_ptr(p) for p in pres])
    x_arr = (P * n)(*[_ptr(x) for x in keep])
    y_arr = (P * n)(*[_ptr(y) for y in ys])
    L = _lib.lib()
    ws = torch.zeros(max(L.endor_cuda_workspace_bytes_batch(views, n), 256), dtype=torch.uint8, device=dev)
    check(L.endor_cuda_gemv_compressed_batch(views, pre_arr, x_arr, y_arr, None, n, ws.data_ptr(), ws.numel(),
                                             _stream_ptr(dev)))
    sync_status(ws, dev)
    return ys


def quantize_values(t: EndorTensor) -> EndorTensor:
    """codec.hpp:306-331 on the device: f16 packed values -> i8 + scale (the
    bitmap is shared, not copied)."""
    if t.dtype != Dtype.F16:
        raise InvalidArgument("quantize_values requires an f16 tensor")
    dev = t.device
    q = _alloc(t.nnz(), dev)
    scale = C.c_float(0.0)
    ws = workspace(1, dev)
    vals = t.values
    if vals.numel() and _ptr(vals) % 2:  # the kernel reads f16 words: realign on the device
        vals = _alloc(vals.numel(), dev).copy_(vals)
    check(_lib.lib().endor_cuda_quantize_values(_ptr(vals), t.nnz(), _ptr(q), C.byref(scale), ws.data_ptr(),
                                                ws.numel(), _stream_ptr(dev)))
    return EndorTensor(t.rows, t.cols, Dtype.I8, t.bitmap, q, quant_scale=scale.value,
                       negative_zero_collapsed=t.negative_zero_collapsed(), validate=False, nnz=t.nnz())


def dequantize_values(t: EndorTensor) -> EndorTensor:
    """codec.hpp:334-349 on the device: i8 packed values + scale -> f16 values
    (bit-exact f32_to_f16 RNE); the bitmap is shared.  decompress_dequant fuses
    this with the expand."""
    if t.dtype != Dtype.I8 or t.quant_scale is None:
        raise InvalidArgument("dequantize_values requires a quantized i8 tensor")
    dev = t.device
    out = _alloc(t.nnz() * 2, dev)
    check(_lib.lib().endor_cuda_dequantize_values(_ptr(t.values), t.nnz(), float(t.quant_scale), _ptr(out),
                                                  _stream_ptr(dev)))
    return EndorTensor(t.rows, t.cols, Dtype.F16, t.bitmap, out,
                       negative_zero_collapsed=t.negative_zero_collapsed(), validate=False, nnz=t.nnz())


VCODE_HEADER_BYTES = 256  # endor_vcode_header


def encode_values(values: torch.Tensor, k_max: int = 0, pin: bool = True) -> torch.Tensor:
    """Lossless transport coding of packed f16 values (vcode.cu; no reference
    counterpart): low bytes raw, high bytes as k-bit dictionary codes plus an
    exception list (k_max 1..7), or -- k_max 0, automatic -- a chunked
    canonical Huffman stream of the high bytes when that is smaller.  ``values`` is the uint8 view of the packed f16 values
    (host or device); returns the blob as a (pinned) host uint8 tensor.  An
    offline, load-time step, like ``compress``.  The blob can be larger than
    the raw values (incompressible high bytes): ship it only when smaller."""
    v = values.reshape(-1).view(torch.uint8)
    if v.numel() % 2:
        raise InvalidArgument("f16 values must hold an even number of bytes")
    v = v.cpu().contiguous()
    nnz = v.numel() // 2
    L = _lib.lib()
    need = C.c_size_t(0)
    check(L.endor_values_encode(_ptr(v), nnz, k_max, None, 0, C.byref(need)))
    blob = torch.empty(need.value, dtype=torch.uint8, pin_memory=pin)
    check(L.endor_values_encode(_ptr(v), nnz, k_max, blob.data_ptr(), blob.numel(), C.byref(need)))
    return blob


def vcode_info(blob: torch.Tensor) -> dict:
    """Header fields of a coded-values blob (host tensor)."""
    h = blob[:VCODE_HEADER_BYTES].numpy()
    u32, u64 = h[:8].view("<u4"), h[8:56].view("<u8")
    mode = "huffman" if int(u32[0]) == 0x31485645 else "fixed"
    return {"mode": mode, "k": int(u32[1]), "nnz": int(u64[0]), "n_exc": int(u64[1]), "blob_bytes": int(u64[5])}


def decode_values(blob: torch.Tensor, device=None) -> torch.Tensor:
    """Decode a coded-values blob on the GPU: returns the packed f16 values as
    a device uint8 tensor (bit-exact with the values that were encoded)."""
    dev = _dev(device)
    hb = blob[:VCODE_HEADER_BYTES].cpu().contiguous()
    L = _lib.lib()
    check(L.endor_values_decode_host_check(hb.data_ptr()))
    info = vcode_info(hb)
    bd = _alloc(blob.numel(), dev)
    bd.copy_(blob.reshape(-1).view(torch.uint8))
    out = _alloc(info["nnz"] * 2, dev)
    check(L.endor_cuda_values_decode(hb.data_ptr(), _ptr(bd), _ptr(out), _stream_ptr(dev)))
    torch.cuda.synchronize(dev)
    return out


def _index_list(idx, dev) -> torch.Tensor:
    t = torch.as_tensor(idx, dtype=torch.int64) if not isinstance(idx, torch.Tensor) else idx
    return t.to(device=dev, dtype=torch.int64).contiguous().reshape(-1)


def _extract(t: EndorTensor, idx, by_rows: bool) -> DenseMatrix:
    dev = t.device
    sel = _index_list(idx, dev)
    k = sel.numel()
    out = DenseMatrix.empty(k if by_rows else t.rows, t.cols if by_rows else k, t.dtype, dev)
    ws = workspace(max(t.element_count(), 1), dev)
    v = t.view()
    fn = _lib.lib().endor_cuda_extract_rows if by_rows else _lib.lib().endor_cuda_extract_cols
    check(fn(C.byref(v), _ptr(sel), k, _ptr(out.data), ws.data_ptr(), ws.numel(), _stream_ptr(dev)))
    sync_status(ws, dev)
    return out


def extract_rows(t: EndorTensor, rows) -> DenseMatrix:
    """codec.hpp:239-266: whole rows (sorted, unique) without materialising W."""
    return _extract(t, rows, True)


def extract_cols(t: EndorTensor, cols) -> DenseMatrix:
    """codec.hpp:271-297: whole columns (sorted, unique)."""
    return _extract(t, cols, False)


class BatchPlan:
    """A prepared batch decompress of up to 64 same-dtype tensors (e.g. one
    decoder layer's weights): two kernel launches for the whole batch."""

    def __init__(self, tensors, outs=None, indices=None):
        """indices: optional RankIndex per tensor (decompress_chunked,
        codec.hpp:205); chunk size 1024 makes the batch a single expand
        launch with no counting pass."""
        if not tensors:
            raise InvalidArgument("empty batch")
        self.tensors = list(tensors)
        dev = self.tensors[0].device
        self.outs = list(outs) if outs is not None else [
            DenseMatrix.empty(t.rows, t.cols, t.dtype, dev) for t in self.tensors]
        n = len(self.tensors)
        self._views = (TensorView * n)(*[t.view() for t in self.tensors])
        self._outs = (C.c_void_p * n)(*[_ptr(o.data) for o in self.outs])
        self.indices = None
        if indices is not None:
            cs = {i.chunk_size for i in indices}
            if len(cs) != 1:
                raise InvalidArgument("one chunk size per batch")
            self.chunk_size = cs.pop()
            for t, i in zip(self.tensors, indices):  # check_index coverage (codec.hpp:174-176)
                want = 0 if t.element_count() == 0 else -(-t.element_count() // self.chunk_size)
                if i.chunk_count() != want:
                    raise CorruptionError("rank index does not cover the bitmap")
            self.indices = [i.prefix.to(device=dev, dtype=torch.int64).contiguous() for i in indices]
            self._pre = (C.c_void_p * n)(*[_ptr(p) for p in self.indices])
        need = _lib.lib().endor_cuda_workspace_bytes_batch(self._views, n)
        if need == 0:
            raise InvalidArgument(_lib.lib().endor_cuda_last_error_string().decode())
        self.ws = torch.zeros(need, dtype=torch.uint8, device=dev)
        self.device = dev

    def launch(self, stream_ptr: Optional[int] = None, phase: int = 0) -> None:
        sp = _stream_ptr(self.device) if stream_ptr is None else stream_ptr
        if self.indices is not None:
            if phase == 1:
                return  # no counting pass on the indexed path
            check(_lib.lib().endor_cuda_decompress_chunked_batch(self._views, self._pre, self.chunk_size,
                                                                 self._outs, len(self.tensors),
                                                                 self.ws.data_ptr(), self.ws.numel(), sp))
            return
        check(_lib.lib().endor_cuda_decompress_batch_phase(self._views, self._outs, len(self.tensors), phase,
                                                           self.ws.data_ptr(), self.ws.numel(), sp))

    def sync(self, stream_ptr: Optional[int] = None) -> None:
        sp = _stream_ptr(self.device) if stream_ptr is None else stream_ptr
        check(_lib.lib().endor_cuda_sync_status(self.ws.data_ptr(), sp))


def decompress_batch(tensors, outs=None, indices=None):
    """decompress() of several tensors in one count + one expand launch, or --
    with a 1024-chunk RankIndex per tensor -- decompress_chunked() of all of
    them in a single expand launch."""
    plan = BatchPlan(tensors, outs, indices)
    plan.launch()
    plan.sync()
    return plan.outs


def build_rank_index(bitmap: Bitmap, chunk_size: int) -> RankIndex:
    """bitmap.hpp:117-132 on the device."""
    dev = bitmap.data.device
    n = bitmap.size()
    chunks = 0 if (n == 0 or chunk_size <= 0) else (n + chunk_size - 1) // chunk_size
    prefix = torch.zeros(max(chunks, 1), dtype=torch.int64, device=dev)
    ws = workspace(n, dev)
    check(_lib.lib().endor_cuda_rank_index(_ptr(bitmap.data), n, chunk_size, prefix.data_ptr(), None,
                                           ws.data_ptr(), ws.numel(), _stream_ptr(dev)))
    sync_status(ws, dev)
    return RankIndex(chunk_size, prefix[:chunks])


def _prefix_ptr(idx: RankIndex, dev: torch.device) -> Tuple[Optional[int], torch.Tensor]:
    p = idx.prefix.to(device=dev, dtype=torch.int64).contiguous()
    return (p.data_ptr() if p.numel() else None), p


def decompress_chunked(t: EndorTensor, idx: RankIndex) -> DenseMatrix:
    """codec.hpp:205-216 on the device."""
    dev = t.device
    out = DenseMatrix.empty(t.rows, t.cols, t.dtype, dev)
    ws = workspace(t.element_count(), dev)
    pp, keep = _prefix_ptr(idx, dev)
    v = t.view()
    check(_lib.lib().endor_cuda_decompress_chunked(C.byref(v), idx.chunk_size, pp, idx.chunk_count(),
                                                   _ptr(out.data), ws.data_ptr(), ws.numel(),
                                                   _stream_ptr(dev)))
    sync_status(ws, dev)
    del keep
    return out


def decompress_chunk_into(t: EndorTensor, idx: RankIndex, k: int, dst: torch.Tensor) -> None:
    """codec.hpp:191-201 on the device: dst is the full dense buffer (uint8)."""
    dev = t.device
    ws = workspace(t.element_count(), dev)
    pp, keep = _prefix_ptr(idx, dev)
    v = t.view()
    dst = dst.view(torch.uint8)
    check(_lib.lib().endor_cuda_decompress_chunk_into(C.byref(v), idx.chunk_size, pp,
                                                      idx.chunk_count(), k, _ptr(dst), dst.numel(),
                                                      ws.data_ptr(), ws.numel(), _stream_ptr(dev)))
    sync_status(ws, dev)
    del keep


# ---- synthetic inputs (weight_gen.hpp) ----------------------------------------------

def synth_weight(rows: int, cols: int, seed: int, dtype: Dtype = Dtype.F16, device=None,
                 row0: int = 0, nrows: Optional[int] = None) -> DenseMatrix:
    """weight_gen.hpp:40-55, bit-exact, for rows [row0, row0+nrows)."""
    dev = _dev(device)
    nrows = rows - row0 if nrows is None else nrows
    out = DenseMatrix.empty(nrows, cols, dtype, dev)
    check(_lib.lib().endor_cuda_synth_weight(rows, cols, int(dtype), seed, row0, nrows,
                                             _ptr(out.data), _stream_ptr(dev)))
    return out


def magnitude_prune(w: DenseMatrix, sparsity: float, inplace: bool = False) -> DenseMatrix:
    """weight_gen.hpp:96-113, bit-exact."""
    out = w if inplace else DenseMatrix(w.rows, w.cols, w.dtype, w.data.clone())
    dev = out.data.device
    n = out.element_count
    ws = workspace(n, dev)
    check(_lib.lib().endor_cuda_magnitude_prune(n, int(out.dtype), float(sparsity), _ptr(out.data),
                                                ws.data_ptr(), ws.numel(), _stream_ptr(dev)))
    return out


def gemv(w: DenseMatrix, x: torch.Tensor, out_f32: Optional[torch.Tensor] = None) -> torch.Tensor:
    """y = W x (f16 in, fp32 accumulate/out) through the hand-written kernel."""
    dev = w.data.device
    if w.dtype != Dtype.F16 or x.dtype != torch.float16 or x.numel() != w.cols:
        raise InvalidArgument("gemv needs f16 W [rows, cols] and f16 x [cols]")
    y = out_f32 if out_f32 is not None else torch.empty(w.rows, dtype=torch.float32, device=dev)
    check(_lib.lib().endor_cuda_gemv(w.rows, w.cols, _ptr(w.data), _ptr(x.contiguous()), _ptr(y), None,
                                     _stream_ptr(dev)))
    return y


def gemv_batch(ws_: Sequence[DenseMatrix], xs: Sequence[torch.Tensor]) -> List[torch.Tensor]:
    """y_i = W_i x_i for a batch of dense f16 matrices in one launch."""
    if len(ws_) != len(xs):
        raise InvalidArgument("one x per matrix")
    if not ws_:
        return []
    dev = ws_[0].data.device
    ys, keep = [], []
    for w, x in zip(ws_, xs):
        if w.dtype != Dtype.F16 or x.dtype != torch.float16 or x.numel() != w.cols:
            raise InvalidArgument("gemv_batch needs f16 W [rows, cols] and f16 x [cols]")
        ys.append(torch.empty(w.rows, dtype=torch.float32, device=dev))
        keep.append(x.contiguous())
    n = len(ws_)
    U, P = C.c_uint64, C.c_void_p
    check(_lib.lib().endor_cuda_gemv_batch((U * n)(*[w.rows for w in ws_]), (U * n)(*[w.cols for w in ws_]),
                                           (P * n)(*[_ptr(w.data) for w in ws_]), (P * n)(*[_ptr(x) for x in keep]),
                                           (P * n)(*[_ptr(y) for y in ys]), None, n, _stream_ptr(dev)))
    return ys
