"""Row-block sharding of bitmap-sparse weights across GPUs (north star (c)).

Shard g of G owns rows [g*R//G, (g+1)*R//G) of a rows x cols matrix.  In the
Endor format (bitmap LSB-first in row-major element order, values packed in
the same order; codec.hpp:21-23, bitmap.hpp:14-17) that row block is

  * a contiguous bitmap bit range [r0*C, r1*C) -- byte aligned when C % 8 == 0,
    4-byte aligned (what the kernels require) when C % 32 == 0 (every catalog
    shape: C in {8192, 9216, 28672, 36864});
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


def shard_tensor(t, shard: RowShard):
    """Device view of one row shard of an EndorTensor (codec.EndorTensor):
    bitmap/values are slices of t's device buffers, value offsets come from
    device popcounts of the bitmap prefix."""
    from . import codec as E
    if shard.cols != t.cols:
        raise ValueError("shard/tensor column mismatch")
    b0, b1 = shard.bitmap_byte_range()
    eb = E.elem_bytes(t.dtype)

    def rank(bit):
        if bit == 0:
            return 0
        return E.Bitmap(bit, data=t.bitmap.data[: (bit + 7) // 8]).count() if bit % 8 == 0 else None

    v0, v1 = rank(shard.bit_begin), rank(shard.bit_end)
    bm = E.Bitmap(shard.bit_end - shard.bit_begin, data=t.bitmap.data[b0:b1])
    vals = t.values[v0 * eb: v1 * eb]
    return E.EndorTensor(shard.rows, shard.cols, t.dtype, bm, vals, validate=False, nnz=v1 - v0)


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


def all_gather_dense(shard_dense, full_rows: int, group=None):
    """Optional NCCL all-gather of dense row shards into the full matrix on
    every rank (only when one device needs the whole dense W).  Shards must be
    equal-sized (R % world == 0) for all_gather_into_tensor."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty(full_rows * shard_dense.cols * (2 if int(shard_dense.dtype) == 0 else 1),
                      dtype=torch.uint8, device=shard_dense.data.device)
    dist.all_gather_into_tensor(out, shard_dense.data.contiguous(), group=group)
    return out


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
    out = torch.empty(width * world, dtype=y_shard.dtype, device=y_shard.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return torch.cat([out[g * width: g * width + sh.rows] for g, sh in enumerate(shards)])
