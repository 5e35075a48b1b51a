"""Host-side logic (no GPU): catalog, size law, row sharding, roofline bytes."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_11674_b200 import catalog
from paper_2406_11674_b200 import shard as S


def test_catalog_matches_reference():
    opt = catalog.model_catalog("opt-66b")
    assert opt.num_layers == 64 and [o.name for o in opt.ops][-2:] == ["fc1", "fc2"]
    assert opt.bytes_per_layer == 2_038_431_744
    llama = catalog.model_catalog("llama2-70b")
    assert llama.num_layers == 80 and catalog.find_op(llama, "attn.k_proj").rows == 1024
    with pytest.raises(ValueError):
        catalog.model_catalog("gpt-5")
    with pytest.raises(ValueError):
        catalog.find_op(opt, "nope")


def test_size_law_and_roofline_bytes():
    from paper_2406_11674_b200 import codec as E
    assert E.compression_ratio(E.Dtype.F16, 0.5) == 0.5625
    assert E.compression_ratio(E.Dtype.I8, 0.5) == 0.625
    assert E.compression_ratio(E.Dtype.F16, 1.0) == 0.0625
    with pytest.raises(E.InvalidArgument):
        E.compression_ratio(E.Dtype.F16, 1.5)
    assert E.endor_values_bytes(E.Dtype.F16, 9216 * 36864 // 2) == 339_738_624
    assert E.endor_bitmap_bytes(9216, 36864) == 42_467_328
    with pytest.raises(E.SizeError):
        E.checked_element_count(1 << 40, 1 << 40)
    # fc1 @50%: 1,061,683,200 algorithmic bytes
    n = 9216 * 36864
    assert catalog.algorithmic_bytes(n, catalog.pruned_nnz(n, 0.5)) == 1_061_683_200
    # OPT layer: 1,146,617,856 compressed bytes
    comp = sum((o.element_count + 7) // 8 + catalog.pruned_nnz(o.element_count, 0.5) * 2
               for o in catalog.model_catalog("opt-66b").ops)
    assert comp == 1_146_617_856


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_row_shards_tile_the_matrix(world):
    rows, cols = 37, 96
    shards = S.row_shards(rows, cols, world)
    assert shards[0].r0 == 0 and shards[-1].r1 == rows
    assert all(a.r1 == b.r0 for a, b in zip(shards, shards[1:]))
    w = O.random_dense(rows, cols, 2, 11, 0.5)
    bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
    got = []
    for sh in shards:
        sb, sv, snnz = S.host_shard_slices(bm, vals, 2, sh)
        st, dense = O.decompress(sh.rows, cols, 2, sb, sv, snnz)
        assert st == 0
        got.append(dense)
    assert np.concatenate(got).tobytes() == w.tobytes()


def test_shard_alignment_rules():
    sh = S.row_shard(9216, 36864, 3, 8)
    b0, b1 = sh.bitmap_byte_range()
    assert b0 % 4 == 0 and (b1 - b0) == sh.rows * 36864 // 8
    with pytest.raises(ValueError):
        S.row_shard(10, 12, 1, 2).bitmap_byte_range()
    with pytest.raises(ValueError):
        S.row_shards(10, 8, 0)


def test_host_rank_matches_oracle():
    w = O.random_dense(50, 40, 2, 3, 0.3)
    bm, _, _, _ = O.compress(w, 50, 40, 2)
    for end in (0, 1, 7, 8, 9, 63, 64, 65, 1000, 2000):
        assert S.host_rank(bm, end) == O.lib().or_rank_range(bm, 0, end)


def test_crc32_combine_matches_zlib():
    import zlib
    rng = np.random.default_rng(5)
    for la, lb in ((0, 0), (1, 0), (0, 7), (13, 1), (1000, 4097), (65536, 3)):
        a = rng.integers(0, 256, la, dtype=np.uint8).tobytes()
        b = rng.integers(0, 256, lb, dtype=np.uint8).tobytes()
        assert S.crc32_combine(zlib.crc32(a), zlib.crc32(b), lb) == zlib.crc32(a + b)
    # a matrix split into row shards, combined in order
    m = rng.integers(0, 256, (37, 64), dtype=np.uint8)
    c = 0
    for sh in S.row_shards(37, 32, 5):
        part = m[sh.r0:sh.r1].tobytes()
        c = S.crc32_combine(c, zlib.crc32(part), len(part))
    assert c == zlib.crc32(m.tobytes())


def test_bit_slice_repacks_any_offset():
    """shard._bit_slice (rows whose bit range is not byte aligned, cols % 8 != 0):
    bits [b0, b1) re-packed LSB-first from bit 0 with zero padding bits."""
    import numpy as np
    import torch
    from paper_2406_11674_b200 import shard as S
    rng = np.random.default_rng(3)
    raw = rng.integers(0, 256, 200, dtype=np.uint8)
    bits = np.unpackbits(raw, bitorder="little")
    for b0, b1 in [(0, 0), (0, 13), (3, 3), (5, 77), (8, 64), (13, 1599), (1590, 1600), (7, 8)]:
        got = S._bit_slice(torch.from_numpy(raw), b0, b1).numpy()
        want = np.packbits(bits[b0:b1], bitorder="little")
        assert got.tobytes() == want.tobytes(), (b0, b1)


def test_row_shards_cover_rows_exactly():
    from paper_2406_11674_b200 import shard as S
    for rows, world in [(1, 8), (5, 8), (9216, 8), (1023, 3)]:
        sh = S.row_shards(rows, 7, world)
        assert sh[0].r0 == 0 and sh[-1].r1 == rows
        assert all(a.r1 == b.r0 for a, b in zip(sh, sh[1:]))
