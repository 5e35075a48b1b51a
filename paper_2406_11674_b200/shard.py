"""Row-block sharding of bitmap-sparse weights across GPUs (north star (c)).

Shard g of G owns rows [g*R//G, (g+1)*R//G) of a rows x cols matrix.  In the
Endor format (bitmap LSB-first in row-major element order, values packed in
the same order; codec.hpp:21-23, bitmap.hpp:14-17) that row block is

  * a contiguous bitmap bit range [r0*C, r1*C) -- byte aligned when C % 8 == 0,
    4-byte aligned (what the kernels require) when C % 32 == 0 (every catalog
    shape: C in {8192, 9216, 28672, 36864}); other widths are re-packed;
  * a contiguous values range [rank(r0*C), rank(r1*C)), rank = Bitmap::rank
    (bitmap.hpp:41).

So each GPU transfers and decompresses its own slice with no inter-GPU
dependency; an NCCL all-gather is needed only when one
device wants the full dense matrix (``all_gather_dense``).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np


@dataclass(frozen=True)
class RowShard:
    rank: int
    world: int
    r0: int
    r1: int
    cols: int

    @property
    def rows(self) -> int:
        return self.r1 - self.r0

    @property
    def bit_begin(self) -> int:
        return self.r0 * self.cols

    @property
    def bit_end(self) -> int:
        return self.r1 * self.cols

    def bitmap_byte_range(self) -> Tuple[int, int]:
        if self.cols % 8:
            raise ValueError("row shards need cols % 8 == 0 to be byte-aligned bitmap slices")
        return self.bit_begin // 8, (self.bit_end + 7) // 8


def row_shards(rows: int, cols: int, world: int) -> List[RowShard]:
    if world < 1:
        raise ValueError("world size must be >= 1")
    return [RowShard(g, world, g * rows // world, (g + 1) * rows // world, cols) for g in range(world)]


def row_shard(rows: int, cols: int, rank: int, world: int) -> RowShard:
    return row_shards(rows, cols, world)[rank]


def host_rank(bitmap: np.ndarray, end_bit: int) -> int:
    """Bitmap::rank(end) on a host LSB-first byte array (planning/tests)."""
    full, rem = divmod(end_bit, 8)
    bits = np.unpackbits(np.asarray(bitmap[:full], dtype=np.uint8), bitorder="little").sum(dtype=np.int64)
    if rem:
        bits += bin(int(bitmap[full]) & ((1 << rem) - 1)).count("1")
    return int(bits)


def host_shard_slices(bitmap: np.ndarray, values: np.ndarray, eb: int, shard: RowShard):
    """(bitmap bytes, values bytes, nnz) of one row shard of a host tensor."""
    b0, b1 = shard.bitmap_byte_range()
    v0 = host_rank(bitmap, shard.bit_begin)
    v1 = host_rank(bitmap, shard.bit_end)
    return bitmap[b0:b1], values[v0 * eb: v1 * eb], v1 - v0


def device_rank(bitmap, bit: int) -> int:
    """Bitmap::rank(bit) (bitmap.hpp:41) of a device bitmap (codec.Bitmap):
    the device popcount of the whole bytes below `bit` plus the low bits of
    the byte it falls in."""
    import torch
    from . import codec as E
    if bit < 0 or bit > bitmap.size():
        raise E.BoundsError("rank position past the bitmap")
    full, rem = divmod(bit, 8)
    r = E.Bitmap(full * 8, data=bitmap.data[:full]).count() if full else 0
    if rem:
        r += int(torch.bitwise_and(bitmap.data[full], (1 << rem) - 1).item()).bit_count()
    return r


def _bit_slice(data, b0: int, b1: int):
    """Bits [b0, b1) of an LSB-first device byte array, re-packed from bit 0
    (zero padding bits), for row shards whose bit range is not byte aligned."""
    import torch
    n = b1 - b0
    lo, hi = b0 // 8, (b1 + 7) // 8
    sh = torch.arange(8, device=data.device, dtype=torch.uint8)
    bits = ((data[lo:hi].unsqueeze(1) >> sh) & 1).reshape(-1)[b0 - 8 * lo: b0 - 8 * lo + n]
    pad = (-n) % 8
    if pad:
        bits = torch.cat([bits, torch.zeros(pad, dtype=torch.uint8, device=data.device)])
    return (bits.reshape(-1, 8) << sh).sum(dim=1, dtype=torch.uint8) if n else bits[:0]


def shard_tensor(t, shard: RowShard, copy: bool = False):
    """One row shard of a device EndorTensor (codec.EndorTensor): its bitmap
    bit range [r0*C, r1*C) and its values [rank(r0*C), rank(r1*C))
    (bitmap.hpp:41, codec.hpp:21-23), sliced out of the whole compressed
    tensor -- never recompressed.

    copy=False returns views into t's buffers where the kernels accept them
    (bitmap byte-aligned and 4-byte aligned; a view that is not 16-byte
    aligned runs the plain fallback expand); copy=True (or a bit range that is
    not byte aligned) gives the shard its own buffers, as a per-GPU transfer
    of the slice would."""
    from . import codec as E
    if shard.cols != t.cols:
        raise ValueError("shard/tensor column mismatch")
    eb = E.elem_bytes(t.dtype)
    b0, b1 = shard.bit_begin, shard.bit_end
    v0 = device_rank(t.bitmap, b0)
    v1 = device_rank(t.bitmap, b1)
    nbytes = (b1 - b0 + 7) // 8
    byte_ok = b0 % 8 == 0
    if byte_ok and not copy and (t.bitmap.data.data_ptr() + b0 // 8) % 4 == 0:
        bm_data = t.bitmap.data[b0 // 8: b0 // 8 + nbytes]
        if (b1 - b0) % 8:  # the last byte also holds the next shard's bits: clear them
            bm_data = bm_data.clone()
            bm_data[-1] &= (1 << ((b1 - b0) % 8)) - 1
        vals = t.values[v0 * eb: v1 * eb]
    else:
        bm_data = E._alloc(nbytes, t.device)
        bm_data.copy_(_bit_slice(t.bitmap.data, b0, b1) if not byte_ok or (b1 - b0) % 8
                      else t.bitmap.data[b0 // 8: b0 // 8 + nbytes])
        vals = E._alloc((v1 - v0) * eb, t.device)
        vals.copy_(t.values[v0 * eb: v1 * eb])
    bm = E.Bitmap(b1 - b0, data=bm_data)
    return E.EndorTensor(shard.rows, shard.cols, t.dtype, bm, vals, validate=False, nnz=v1 - v0,
                         negative_zero_collapsed=t.negative_zero_collapsed())


def _gf2_times(mat: List[int], vec: int) -> int:
    s, i = 0, 0
    while vec:
        if vec & 1:
            s ^= mat[i]
        vec >>= 1
        i += 1
    return s


def crc32_combine(crc1: int, crc2: int, len2: int) -> int:
    """CRC-32 (zlib) of A || B from crc(A), crc(B) and len(B): lets every rank
    checksum its own row shard and rank 0 assemble the whole matrix's CRC
    (compared with the reference's, tests/golden/large.json) without moving
    the shards.  zlib's crc32_combine: apply len2 zero bytes to crc1 by
    repeated squaring of the GF(2) shift operator."""
    if len2 <= 0:
        return crc1
    odd = [0xEDB88320] + [1 << n for n in range(31)]  # operator for one zero bit
    even = [_gf2_times(odd, odd[n]) for n in range(32)]  # two bits
    odd = [_gf2_times(even, even[n]) for n in range(32)]  # four bits
    while True:
        even = [_gf2_times(odd, odd[n]) for n in range(32)]
        if len2 & 1:
            crc1 = _gf2_times(even, crc1)
        len2 >>= 1
        if not len2:
            break
        odd = [_gf2_times(even, even[n]) for n in range(32)]
        if len2 & 1:
            crc1 = _gf2_times(odd, crc1)
        len2 >>= 1
        if not len2:
            break
    return (crc1 ^ crc2) & 0xFFFFFFFF


def _gather_into(out, inp, group):
    """all_gather_into_tensor; under gloo (CPU collectives, e.g. ranks sharing
    one GPU) CUDA buffers are staged through host memory."""
    import torch.distributed as dist
    if out.is_cuda and dist.get_backend(group) == "gloo":
        o = out.cpu()
        dist.all_gather_into_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp, group=group)
    return out


def all_gather_dense(shard_dense, full_rows: int, group=None):
    """Optional all-gather (NCCL over NVLink) of dense row shards into the full
    matrix on every rank -- only when one device needs the whole dense W
    (SURVEY.md 8(e)).  Ragged shards (R % world != 0) are padded to the largest
    shard for the collective and trimmed after.  Returns uint8 row-major bytes."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    row_bytes = shard_dense.cols * (2 if int(shard_dense.dtype) == 0 else 1)
    shards = row_shards(full_rows, 1, world)
    width = max(sh.rows for sh in shards) * row_bytes
    dev = shard_dense.data.device
    mine = shard_dense.data.reshape(-1)
    if mine.numel() != width:
        buf = torch.zeros(width, dtype=torch.uint8, device=dev)
        buf[: mine.numel()] = mine
        mine = buf
    out = _gather_into(torch.empty(width * world, dtype=torch.uint8, device=dev), mine.contiguous(), group)
    if all(sh.rows * row_bytes == width for sh in shards):
        return out
    return torch.cat([out[g * width: g * width + sh.rows * row_bytes] for g, sh in enumerate(shards)])


def all_gather_y(y_shard, full_rows: int, group=None):
    """Concatenate the row-shard GEMV outputs y_g (rows r0..r1 of y = W x) into
    the full y on every rank (the only exchange a row-sharded
    GEMV ever needs; rows * 4 bytes).  Ragged shards (R % world != 0) are
    padded to the largest shard for the collective and trimmed after."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    shards = row_shards(full_rows, 1, world)
    width = max(sh.rows for sh in shards)
    buf = torch.zeros(width, dtype=y_shard.dtype, device=y_shard.device)
    buf[: y_shard.numel()] = y_shard
    out = _gather_into(torch.empty(width * world, dtype=y_shard.dtype, device=y_shard.device), buf, group)
    return torch.cat([out[g * width: g * width + sh.rows] for g, sh in enumerate(shards)])
