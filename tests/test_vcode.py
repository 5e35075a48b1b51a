"""Coded-values transport (csrc/vcode.cu; no reference counterpart): the blob
format restated in numpy (the checker), the host encoder against it, the GPU
decoder bit-exact against the values that were encoded, and the offload
pipeline with coded ops giving the same y and W as with raw values.

The reference moves the packed values over the link as they are
(sim.hpp:200-204); this coding is lossless, so every check here is bit-exact.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2406_11674_b200 import _lib
from paper_2406_11674_b200 import codec as E


def decode_huff_np(blob: np.ndarray) -> np.ndarray:
    """Huffman mode ("EVH1"): chunks of 512 values, each from its own word
    offset, decoded LSB-first through the blob's 4096-entry table."""
    u64 = blob[8:56].view("<u8")
    nnz, words, lo_off, offs_off, stream_off, nbytes = map(int, u64)
    assert nbytes == blob.size == stream_off + (4 * words + 15) // 16 * 16 and int(blob[4:8].view("<u4")[0]) == 12
    lut = blob[256:256 + 8192].view("<u2")
    lo = blob[lo_off:lo_off + nnz].astype(np.uint16)
    nch = (nnz + 511) // 512
    offs = blob[offs_off:offs_off + 4 * (nch + 1)].view("<u4")
    stream = blob[stream_off:stream_off + 4 * words].view("<u4")
    assert offs[0] == 0 and offs[-1] == words and np.all(np.diff(offs.astype(np.int64)) >= 0)
    hi = np.zeros(nnz, np.uint16)
    for c in range(nch):
        bits = int.from_bytes(stream[offs[c]:offs[c + 1]].tobytes(), "little")
        for i in range(c * 512, min(nnz, c * 512 + 512)):
            e = int(lut[bits & 0xFFF])
            assert e >> 8, "unassigned table entry"
            hi[i] = e & 0xFF
            bits >>= e >> 8
    return (lo | (hi << 8)).astype(np.uint16)


def decode_np(blob: np.ndarray) -> np.ndarray:
    """The blob format of include/endor_cuda.h (endor_vcode_header), restated."""
    u32 = blob[:8].view("<u4")
    u64 = blob[8:56].view("<u8")
    if u32[0] == 0x31485645:
        return decode_huff_np(blob)
    assert u32[0] == 0x31435645
    k, nnz, n_exc, lo_off, code_off, exc_off, nbytes = int(u32[1]), *map(int, u64)
    dic = blob[64:192]
    assert nbytes == blob.size
    lo = blob[lo_off:lo_off + nnz].astype(np.uint16)
    words = np.concatenate([blob[code_off:exc_off].view("<u4").astype(np.uint64), np.zeros(2, np.uint64)])
    bit = np.arange(nnz, dtype=np.uint64) * np.uint64(k)
    wi, sh = bit >> np.uint64(5), bit & np.uint64(31)
    pair = words[wi] | (words[wi + np.uint64(1)] << np.uint64(32))
    code = (pair >> sh) & np.uint64((1 << k) - 1)
    hi = dic[code.astype(np.int64)].astype(np.uint16)
    exc = blob[exc_off:exc_off + 8 * n_exc].view("<u8")
    assert np.all(code[(exc >> np.uint64(8)).astype(np.int64)] == (1 << k) - 1)
    hi[(exc >> np.uint64(8)).astype(np.int64)] = (exc & np.uint64(0xFF)).astype(np.uint16)
    return (lo | (hi << 8)).astype(np.uint16)


def encode(vals_u16: np.ndarray, k_max: int = 0) -> np.ndarray:
    L = _lib.lib()
    v = np.ascontiguousarray(vals_u16.astype(np.uint16))
    need = C.c_size_t(0)
    ptr = v.ctypes.data if v.size else None
    E.check(L.endor_values_encode(ptr, v.size, k_max, None, 0, C.byref(need)))
    out = np.zeros(need.value, np.uint8)
    E.check(L.endor_values_encode(ptr, v.size, k_max, out.ctypes.data, out.size, C.byref(need)))
    return out


def pruned_f16(n: int, seed: int) -> np.ndarray:
    """Surviving values of a magnitude-pruned f16 weight (|w| above the median)."""
    w = np.random.default_rng(seed).standard_normal(2 * n).astype(np.float16) * np.float16(0.02)
    keep = np.abs(w) > np.median(np.abs(w))
    return w[keep][:n].view(np.uint16)


CASES = {
    "empty": np.zeros(0, np.uint16),
    "one": np.array([0x3C00], np.uint16),
    "31": pruned_f16(31, 1),
    "32": pruned_f16(32, 2),
    "33": pruned_f16(33, 3),
    "pruned_1000": pruned_f16(1000, 4),
    "pruned_100k": pruned_f16(100_003, 5),
    "uniform_u16": np.random.default_rng(6).integers(0, 1 << 16, 50_001, dtype=np.uint16),
    "specials": np.array([0x7C00, 0xFC00, 0x7E00, 0x7C01, 0xFFFF, 0x8000, 0x0001, 0x8001] * 37, np.uint16),
    "one_hi_byte": (np.random.default_rng(7).integers(0, 256, 4097, dtype=np.uint16) | 0x3A00).astype(np.uint16),
    # geometric high bytes: Huffman lengths past 12 bits, flattened to fit the table
    "geometric": ((np.minimum(np.random.default_rng(8).geometric(0.5, 70_001) - 1, 40).astype(np.uint16) + 0x30) << 8
                  | np.random.default_rng(9).integers(0, 256, 70_001, dtype=np.uint16)).astype(np.uint16),
}


@pytest.mark.parametrize("k_max", [0, 7])
@pytest.mark.parametrize("name", sorted(CASES))
def test_encode_round_trip_numpy(name, k_max):
    v = CASES[name]
    blob = encode(v, k_max)
    assert np.array_equal(decode_np(blob), v)


def test_huffman_code_lengths_are_limited_to_the_table():
    # geometric high-byte frequencies (2^-1, 2^-2, ...): an unbounded Huffman code
    # would go past 12 bits; the lengths are flattened until they fit the table
    rng = np.random.default_rng(21)
    hi = np.minimum(rng.geometric(0.5, 400_000) - 1, 40).astype(np.uint16)
    v = ((hi + 0x30) << 8 | rng.integers(0, 256, hi.size, dtype=np.uint16)).astype(np.uint16)
    blob = encode(v, 0)
    assert int(blob[:4].view("<u4")[0]) == 0x31485645
    lut = blob[256:256 + 8192].view("<u2")
    assert (lut >> 8).max() <= 12 and (lut >> 8).min() >= 1  # every entry assigned, no code past 12 bits
    assert len(np.unique(hi)) > 13  # more symbols than a 12-bit chain of halvings could hold
    assert np.array_equal(decode_np(blob), v)


def test_automatic_mode_picks_the_smaller_blob():
    for name, v in CASES.items():
        auto, fixed = encode(v, 0), encode(v, 7)
        assert auto.size <= fixed.size, name
    v = CASES["pruned_100k"]
    assert int(encode(v, 0)[:4].view("<u4")[0]) == 0x31485645  # Huffman wins on pruned weights


@pytest.mark.parametrize("k_max", [1, 2, 3, 5, 7])
def test_k_max_bounds_code_width(k_max):
    v = CASES["uniform_u16"]
    blob = encode(v, k_max)
    assert 1 <= int(blob[4:8].view("<u4")[0]) <= k_max
    assert np.array_equal(decode_np(blob), v)


def test_pruned_weights_shrink():
    # the high byte of pruned (Gaussian) weights is low-entropy: the blob beats 2 B per value
    v = CASES["pruned_100k"]
    blob = encode(v, 7)
    assert blob.size < 0.85 * 2 * v.size
    assert int(blob[4:8].view("<u4")[0]) <= 6
    assert encode(v).size < encode(v, 7).size  # Huffman: near the high byte entropy (3.95 bits here) + an 8 KiB table


def test_single_high_byte_is_one_bit_without_exceptions():
    v = CASES["one_hi_byte"]
    blob = encode(v, 7)
    u64 = blob[8:56].view("<u8")
    assert int(blob[4:8].view("<u4")[0]) == 1 and int(u64[1]) == 0


def test_header_check_and_arguments():
    L = _lib.lib()
    blob = encode(CASES["pruned_1000"])
    assert L.endor_values_decode_host_check(blob.ctypes.data) == 0
    for off, val in ((0, 0x00), (4, 9), (8, 0xFF), (40, 0x01)):  # magic, k, nnz, exc_off
        bad = blob.copy()
        bad[off] ^= val if val else 0x55
        assert L.endor_values_decode_host_check(bad.ctypes.data) == 2  # CORRUPTION
    need = C.c_size_t(0)
    v = CASES["pruned_1000"]
    assert L.endor_values_encode(v.ctypes.data, v.size, -1, None, 0, C.byref(need)) == 4
    assert L.endor_values_encode(v.ctypes.data, v.size, 8, None, 0, C.byref(need)) == 4
    hb = encode(CASES["pruned_100k"])  # Huffman header: recomputed offsets too
    assert L.endor_values_decode_host_check(hb.ctypes.data) == 0
    for off in (4, 16, 40):  # LUT width, stream words, stream offset
        bad = hb.copy()
        bad[off] ^= 0x01
        assert L.endor_values_decode_host_check(bad.ctypes.data) == 2
    small = np.zeros(16, np.uint8)
    assert L.endor_values_encode(v.ctypes.data, v.size, 7, small.ctypes.data, small.size, C.byref(need)) == 4


# ---- GPU: the decoder and the pipeline ----------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("k_max", [0, 7])
@pytest.mark.parametrize("name", sorted(CASES))
def test_gpu_decode_bit_exact(name, k_max):
    v = CASES[name]
    blob = torch.from_numpy(encode(v, k_max))
    out = E.decode_values(blob)
    assert np.array_equal(out.cpu().numpy().view(np.uint16), v)


@pytest.mark.gpu
@pytest.mark.parametrize("k_max", [0, 1, 3, 7])
def test_gpu_decode_large_with_exceptions(k_max):
    rng = np.random.default_rng(11)
    v = pruned_f16((1 << 22) + 5, 12)
    v[rng.integers(0, v.size, 5000)] = rng.integers(0, 1 << 16, 5000, dtype=np.uint16)  # rare high bytes
    blob = torch.from_numpy(encode(v, k_max))
    assert E.vcode_info(blob)["n_exc"] > 0  # exceptions (fixed k) / stream words (Huffman)
    assert np.array_equal(E.decode_values(blob).cpu().numpy().view(np.uint16), v)


@pytest.mark.gpu
def test_gpu_encode_values_of_synth_layer():
    dev = torch.device("cuda", 0)
    w = E.synth_weight(512, 4096, 7, device=dev)
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    blob = E.encode_values(t.values)
    assert blob.is_pinned() and blob.numel() < 0.8 * t.values.numel()
    assert torch.equal(E.decode_values(blob).cpu(), t.values.cpu())


@pytest.mark.gpu
def test_gpu_pipeline_coded_ops_match_raw():
    from paper_2406_11674_b200.pipeline import HostOp, OffloadPipeline, pinned_copy
    dev = torch.device("cuda", 0)
    ops_raw, ops_coded, ts = [], [], []
    for i, (r, c) in enumerate([(1024, 2048), (768, 3072), (1000, 1030)]):
        w = E.synth_weight(r, c, 100 + i, device=dev)
        E.magnitude_prune(w, 0.5, inplace=True)
        t = E.compress(w)
        ts.append(t)
        g = torch.Generator(device="cpu").manual_seed(i)
        x = ((torch.rand(c, generator=g) * 2 - 1).half()).to(dev)
        bm, vals = pinned_copy(t.bitmap.data), pinned_copy(t.values)
        for lst, vc in ((ops_raw, None), (ops_coded, E.encode_values(t.values))):
            lst.append(HostOp(r, c, 0, bm, vals if vc is None else torch.empty(0, dtype=torch.uint8), t.nnz(),
                              x=x, y=torch.empty(r, dtype=torch.float32, device=dev),
                              dense=torch.empty(r * c * 2, dtype=torch.uint8, device=dev), vcode=vc))
    pipe = OffloadPipeline(0, 1024 * 3072, ring_depth=2)
    pipe.run(ops_raw, sync=True)
    pipe.run(ops_coded, sync=True)
    st = pipe.stats()
    assert st["h2d_bytes"] == sum(o.compressed_bytes for o in ops_coded)
    assert st["h2d_bytes"] < sum(o.compressed_bytes for o in ops_raw)
    for a, b, t in zip(ops_raw, ops_coded, ts):
        assert torch.equal(a.y, b.y)  # same values -> same GEMV, bit for bit
        assert torch.equal(a.dense, b.dense)
        ref = E.decompress(t)
        assert torch.equal(b.dense, ref.data[: t.rows * t.cols * 2])
    # fused decompress -> GEMV path (no dense_dev) for both
    for o in ops_raw + ops_coded:
        o.dense = None
    pipe.run(ops_raw, sync=True)
    y_ref = [o.y.clone() for o in ops_raw]
    pipe.run(ops_coded, sync=True)
    for yr, o in zip(y_ref, ops_coded):
        assert torch.equal(yr, o.y)
    pipe.close()


@pytest.mark.gpu
def test_gpu_pipeline_rejects_bad_blob():
    from paper_2406_11674_b200.pipeline import HostOp, OffloadPipeline, pinned_copy
    dev = torch.device("cuda", 0)
    w = E.synth_weight(256, 1024, 3, device=dev)
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    blob = E.encode_values(t.values)
    blob[0] ^= 1
    op = HostOp(256, 1024, 0, pinned_copy(t.bitmap.data), torch.empty(0, dtype=torch.uint8), t.nnz(), vcode=blob)
    pipe = OffloadPipeline(0, 256 * 1024)
    with pytest.raises(E.CorruptionError):
        pipe.run([op], sync=True)
    blob[0] ^= 1
    op.nnz = t.nnz() - 1  # blob and op disagree
    with pytest.raises(E.InvalidArgument):
        pipe.run([op], sync=True)
    pipe.close()
