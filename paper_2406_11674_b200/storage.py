""".endor containers to and from the GPU (the reference's
file_io.hpp:187-277, re-targeted at device memory).

``read_endor_file(path, device)`` is ``read_endor_file`` / ``decode_endor``
(file_io.hpp:212-277) with a device-resident result: the header is parsed and
validated on the host, the bitmap and values sections move to the GPU through
cuFile (GPUDirect Storage, or cuFile's compatibility mode when nvidia-fs is
absent) or O_DIRECT reads through pinned bounce buffers, and the CRC /
padding / popcount checks run on the device copy.  ``write_endor_file`` is the
byte-identical encoder (file_io.hpp:187-210).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import torch

from . import _lib
from .codec import Bitmap, Dtype, EndorTensor, _dev, _stream_ptr, check, encode_values, workspace

MODES = {0: "auto", 1: "gds", 2: "cufile-compat", 3: "posix-odirect"}


def probe(path: str) -> _lib.FileInfo:
    """Header + layout validation in decode_endor's order (FormatError kinds)."""
    info = _lib.FileInfo()
    check(_lib.lib().endor_file_probe(os.fsencode(path), C.byref(info)))
    return info


def encode_endor(t: EndorTensor, version: int = 1) -> bytes:
    """encode_endor (file_io.hpp:187-210): byte-identical container bytes
    (version 2: the same container with 4 KiB-aligned sections, for GDS;
    version 3: v2 with the f16 values as a lossless coded-values blob, which
    the reader decodes on the GPU -- fewer bytes from storage)."""
    bm = t.bitmap.to_bytes()
    flags = (1 if t.quant_scale is not None else 0) | (2 if t.negative_zero_collapsed() else 0)
    L = _lib.lib()
    if version == 3:
        if t.dtype != Dtype.F16 or t.quant_scale is not None:
            raise ValueError("a v3 container holds coded f16 values")
        blob = encode_values(t.values, pin=False).numpy().tobytes()
        args3 = (t.rows, t.cols, flags, bm, blob, t.nnz())
        n = L.endor_file_encode_v3(*args3, None, 0)
        buf = C.create_string_buffer(n)
        if n == 0 or L.endor_file_encode_v3(*args3, buf, n) != n:
            raise ValueError("cannot encode this tensor")
        return buf.raw
    vals = t.values.cpu().numpy().tobytes()
    args = (t.rows, t.cols, int(t.dtype), flags, float(t.quant_scale or 0.0), bm, vals, t.nnz())
    enc = {1: L.endor_file_encode, 2: L.endor_file_encode_v2}[version]
    n = enc(*args, None, 0)
    buf = C.create_string_buffer(n)
    if n == 0 or enc(*args, buf, n) != n:
        raise ValueError("cannot encode this tensor")
    return buf.raw


def write_endor_file(t: EndorTensor, path: str, version: int = 1) -> int:
    data = encode_endor(t, version)
    with open(path, "wb") as f:
        f.write(data)
    return len(data)


class Reader:
    """An endor_reader: cuFile / POSIX transfer engine bound to one device."""

    def __init__(self, device=None, mode: int = 0, bounce_bytes: int = 64 << 20):
        self.device = _dev(device)
        h = C.c_void_p()
        check(_lib.lib().endor_reader_create(self.device.index or 0, bounce_bytes, mode, C.byref(h)))
        self._h = h

    @property
    def mode(self) -> str:
        return MODES[_lib.lib().endor_reader_mode(self._h)]

    def stats(self):
        s, b = C.c_double(), C.c_uint64()
        check(_lib.lib().endor_reader_stats(self._h, C.byref(s), C.byref(b)))
        return s.value, b.value

    def read(self, path: str, verify: bool = True, info: Optional[_lib.FileInfo] = None) -> EndorTensor:
        info = info if info is not None else probe(path)
        dev = self.device
        n = info.rows * info.cols
        bm = torch.zeros(((info.bitmap_bytes + 15) // 16) * 16 + 16, dtype=torch.uint8, device=dev)
        nvals = info.values_out_bytes  # v3: the decoded f16 values, not the coded section
        vals = torch.empty(max(nvals, 1) + 16, dtype=torch.uint8, device=dev)
        ws = workspace(max(n, 1), dev)
        check(_lib.lib().endor_reader_read(self._h, os.fsencode(path), C.byref(info), bm.data_ptr(),
                                           vals.data_ptr(), 1 if verify else 0, ws.data_ptr(), ws.numel(),
                                           _stream_ptr(dev)))
        dt = Dtype(info.dtype)
        return EndorTensor(info.rows, info.cols, dt, Bitmap(n, data=bm[: info.bitmap_bytes]),
                           vals[:nvals],
                           quant_scale=info.quant_scale if info.flags & 1 else None,
                           negative_zero_collapsed=bool(info.flags & 2), validate=False, nnz=info.nnz)

    def close(self) -> None:
        if self._h:
            _lib.lib().endor_reader_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def read_endor_file(path: str, device=None, verify: bool = True, mode: int = 0) -> EndorTensor:
    """read_endor_file (file_io.hpp:274-277) into device memory."""
    r = Reader(device, mode)
    try:
        return r.read(path, verify)
    finally:
        r.close()
