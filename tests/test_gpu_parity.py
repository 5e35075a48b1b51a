"""GPU parity: the sm_100a path (through the C ABI) against the oracle and the
reference's golden vectors.  Bit-exact for every byte/index result.

Ports the assertions of the reference's test_codec.cpp, test_bitmap.cpp,
test_weight_gen.cpp and acceptance.cpp criterion 3 (not the code).
"""
import ctypes as C
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


def crc(b) -> int:
    if isinstance(b, torch.Tensor):
        b = b.cpu().numpy()
    return zlib.crc32(np.ascontiguousarray(b).view(np.uint8).tobytes()) & 0xFFFFFFFF


@pytest.fixture(scope="module")
def E(cuda_lib):
    from paper_2406_11674_b200 import codec
    return codec


def dev_bytes(a, pad=16, offset=0):
    """Upload bytes into a fresh device buffer at a chosen byte offset."""
    a = np.ascontiguousarray(np.asarray(a).view(np.uint8).reshape(-1))
    buf = torch.zeros(a.size + pad + offset + 16, dtype=torch.uint8, device="cuda")
    view = buf[offset: offset + a.size]
    if a.size:
        view.copy_(torch.from_numpy(a.copy()))
    return view


def make_tensor(E, rows, cols, eb, bm, vals, nnz, values_offset=0, validate=True):
    n = rows * cols
    bitmap = E.Bitmap(n, data=dev_bytes(bm) if n else None)
    values = dev_bytes(vals, offset=values_offset)
    dt = E.Dtype.F16 if eb == 2 else E.Dtype.I8
    return E.EndorTensor(rows, cols, dt, bitmap, values, validate=validate, nnz=nnz)


def h(s):
    return np.frombuffer(bytes.fromhex(s), np.uint8)


# ---- KATs (test_codec.cpp / test_bitmap.cpp / test_weight_gen.cpp) ------------

def test_hand_built_2x2(E, kats):
    k = kats["hand_2x2"]
    t = make_tensor(E, 2, 2, 2, h(k["bitmap"]), h(k["values"]), 2)
    out = E.decompress(t)
    assert out.bytes().hex() == k["dense"]


def test_empty_tensor_decompresses_to_zeros(E, kats):
    k = kats["empty_3x3"]
    t = make_tensor(E, 3, 3, 2, h(k["bitmap"]), np.zeros(0, np.uint8), 0)
    assert E.decompress(t).bytes().hex() == k["dense"]


@pytest.mark.parametrize("name", ["nan_inf", "negzero"])
def test_compress_decompress_kats(E, kats, name):
    k = kats[name]
    dense = O.decompress(k["rows"], k["cols"], k["eb"], h(k["bitmap"]), h(k["values"]), k["nnz"])[1]
    t = make_tensor(E, k["rows"], k["cols"], k["eb"], h(k["bitmap"]), h(k["values"]), k["nnz"])
    assert E.decompress(t).bytes().hex() == k["dense"] == dense.tobytes().hex()
    if name == "negzero":
        w = np.array([0x8000, 0xBC00, 0, 0], np.uint16)
        ct = E.compress(E.DenseMatrix.from_host(2, 2, E.Dtype.F16, w.tobytes()))
        assert ct.negative_zero_collapsed() and ct.nnz() == 1
        assert ct.bitmap.to_bytes().hex() == k["bitmap"]


def test_popcount_mismatch_raises_corruption(E, kats):
    k = kats["popcount_mismatch"]
    assert k["status"] == 2
    with pytest.raises(E.CorruptionError):
        make_tensor(E, 2, 2, 2, h(k["bitmap"]), h(k["values"]), 2, validate=True)
    t = make_tensor(E, 2, 2, 2, h(k["bitmap"]), h(k["values"]), 2, validate=False)
    with pytest.raises(E.CorruptionError):
        E.decompress(t)


def test_padding_bits_rejected(E):
    # bitmap.hpp:78-84: bit 10 of a 10-bit bitmap is padding
    t = make_tensor(E, 1, 10, 2, np.array([0x00, 0x06], np.uint8), np.zeros(4, np.uint8), 2,
                    validate=False)
    with pytest.raises(E.CorruptionError):
        E.decompress(t)


def test_checkerboard_size_law(E, kats):
    k = kats["checkerboard"]
    w = np.zeros(128, np.uint16)
    w[::2] = 0x3C00
    t = E.compress(E.DenseMatrix.from_host(8, 16, E.Dtype.F16, w.tobytes()))
    assert t.bitmap.to_bytes().hex() == k["bitmap"]
    assert t.compressed_bytes() / 256 == 0.5625 == k["compressed_bytes"] / k["dense_bytes"]


def test_lsb_first_and_rank_index_kats(E, kats):
    alt = kats["alt_prefix"]
    b = E.Bitmap.from_bytes(h(alt["bitmap"]).tobytes(), 256, device="cuda")
    idx = E.build_rank_index(b, 64)
    assert idx.prefix.cpu().tolist() == alt["prefix"] == [0, 32, 64, 96]
    z = kats["zero_prefix"]
    assert E.build_rank_index(E.Bitmap(300, device="cuda"), 128).prefix.cpu().tolist() == z["prefix"]
    for cs, st in kats["bad_chunk"].items():
        if st:
            with pytest.raises(E.InvalidArgument):
                E.build_rank_index(E.Bitmap(128, device="cuda"), int(cs))


def test_synth_weight_golden(E, kats):
    w = E.synth_weight(4, 4, seed=0, device="cuda")
    assert np.frombuffer(w.bytes(), np.uint16).tolist() == kats["synth_4x4_seed0"]


def test_prune_1x4(E, kats):
    k = kats["prune_1x4"]
    w = E.DenseMatrix.from_host(1, 4, E.Dtype.F16, np.array(k["input"], np.uint16).tobytes())
    p = E.magnitude_prune(w, 0.5)
    assert np.frombuffer(p.bytes(), np.uint16).tolist() == k["output"]


# ---- seeded round trips + chunked + chunk_into -----------------------------------

def test_seeded_cases(E, seeded_cases):
    for c in seeded_cases:
        rows, cols, eb, n = c["rows"], c["cols"], c["eb"], c["rows"] * c["cols"]
        w = O.random_dense(rows, cols, eb, c["seed"], c["zero_fraction"])
        assert crc(w) == c["crc_dense"]
        dt = E.Dtype.F16 if eb == 2 else E.Dtype.I8
        t = E.compress(E.DenseMatrix.from_host(rows, cols, dt, w.tobytes()))
        assert t.nnz() == c["nnz"]
        assert crc(t.bitmap.data) == c["crc_bitmap"] and crc(t.values) == c["crc_values"]
        assert crc(E.decompress(t).data) == c["crc_dense"]
        for cs, pref in c["prefix"].items():
            idx = E.build_rank_index(t.bitmap, int(cs))
            assert idx.prefix.cpu().tolist() == pref
            assert crc(E.decompress_chunked(t, idx).data) == c["crc_dense"]


@pytest.mark.parametrize("offset", [0, 1, 2, 3, 6, 14])
def test_unaligned_values_window(E, offset):
    """values pointer at every byte misalignment (the .endor layout puts the
    values at 32 + ceil(n/8), file_io.hpp:32-36)."""
    for eb, (rows, cols) in [(2, (37, 200)), (1, (16, 100)), (2, (129, 515))]:
        w = O.random_dense(rows, cols, eb, 1234 + offset, 0.55)
        bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
        t = make_tensor(E, rows, cols, eb, bm, vals, nnz, values_offset=offset)
        assert E.decompress(t).bytes() == w.tobytes()


@pytest.mark.parametrize("bm_offset", [4, 8, 12])
def test_bitmap_not_16B_aligned_uses_fallback(E, bm_offset):
    """A bitmap slice that is only 4-byte aligned (e.g. a row shard) takes
    the plain-load expand kernel; results must be identical."""
    for eb, (rows, cols) in [(2, (129, 515)), (1, (77, 300)), (2, (64, 8192 + 64))]:
        w = O.random_dense(rows, cols, eb, 99 + bm_offset, 0.5)
        bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
        n = rows * cols
        bitmap = E.Bitmap(n, data=dev_bytes(bm, offset=bm_offset))
        dt = E.Dtype.F16 if eb == 2 else E.Dtype.I8
        t = E.EndorTensor(rows, cols, dt, bitmap, dev_bytes(vals, offset=3))
        assert E.decompress(t).bytes() == w.tobytes()
        idx = E.build_rank_index(bitmap, 256)
        assert E.decompress_chunked(t, idx).bytes() == w.tobytes()


def test_batch_decompress_matches_oracle(E):
    """One count + one expand launch over mixed tensors (ragged sizes, both
    sparsity extremes, an empty one) == per-tensor oracle decompress."""
    cases = [(37, 200, 0.6), (1, 1, 0.0), (129, 515, 0.5), (64, 8192, 0.0), (3, 5, 1.0),
             (300, 1000, 0.95), (0, 7, 0.5), (512, 1024, 0.3)]
    tensors, wants = [], []
    for i, (r, c, z) in enumerate(cases):
        w = O.random_dense(r, c, 2, 500 + i, z)
        bm, vals, nnz, _ = O.compress(w, r, c, 2)
        tensors.append(make_tensor(E, r, c, 2, bm, vals, nnz, values_offset=i % 3 * 2))
        wants.append(w.tobytes())
    outs = E.decompress_batch(tensors)
    for o, w in zip(outs, wants):
        assert o.bytes() == w
    # a corrupt member (nnz one short) is reported for the whole batch
    bad = tensors[2]
    tensors[2] = E.EndorTensor(bad.rows, bad.cols, bad.dtype, bad.bitmap, bad.values[:-2], validate=False)
    with pytest.raises(E.CorruptionError):
        E.decompress_batch(tensors)


def test_chunked_1024_fast_path(E, seeded_cases):
    """decompress_chunked with a 1024-element RankIndex: one expand launch fed
    by the index (no counting pass), bit-exact; batched over mixed tensors."""
    tensors, idxs, wants = [], [], []
    for i, c in enumerate(seeded_cases[:40]):
        rows, cols, eb = c["rows"], c["cols"], c["eb"]
        if eb != 2:
            continue
        w = O.random_dense(rows, cols, eb, c["seed"], c["zero_fraction"])
        bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
        t = make_tensor(E, rows, cols, eb, bm, vals, nnz, values_offset=(i % 4) * 2)
        idx = E.build_rank_index(t.bitmap, 1024)
        _, ref_p = O.rank_index(bm, rows * cols, 1024)
        assert idx.prefix.cpu().numpy().astype(np.uint64).tolist() == ref_p.tolist()
        assert E.decompress_chunked(t, idx).bytes() == w.tobytes()
        tensors.append(t)
        idxs.append(idx)
        wants.append(w.tobytes())
    for k in range(0, len(tensors), 16):
        outs = E.decompress_batch(tensors[k:k + 16], indices=idxs[k:k + 16])
        assert [o.bytes() for o in outs] == wants[k:k + 16]


def test_chunked_1024_index_errors_are_safe(E):
    rows, cols = 300, 1000
    w = O.random_dense(rows, cols, 2, 31, 0.5)
    bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
    t = make_tensor(E, rows, cols, 2, bm, vals, nnz)
    good = E.build_rank_index(t.bitmap, 1024)
    # last entry wrong -> CorruptionError, as check_index (codec.hpp:179-182)
    bad = good.prefix.clone()
    bad[-1] += 1
    with pytest.raises(E.CorruptionError):
        E.decompress_chunked(t, E.RankIndex(1024, bad))
    # wrong middle entries: check_index (codec.hpp:170-184) only tests the last
    # entry, and so does this one-launch path; an entry that would read outside
    # the tile's staged window is reported, any other yields garbage like the
    # reference -- never an illegal access
    for v in (3, 10 ** 12, -5):
        bad = good.prefix.clone()
        bad[len(bad) // 2] = v if v != 3 else bad[len(bad) // 2] + 3
        try:
            E.decompress_chunked(t, E.RankIndex(1024, bad))
        except E.CorruptionError:
            pass
    # adversarial but validation-passing indices: monotone, <= 1024 values per
    # sub-tile, last entry right -- wrong starts inside / past the windows read
    # garbage (as the reference would) but never outside the staged buffers
    rng = np.random.default_rng(3)
    for trial in range(20):
        bad = good.prefix.clone().cpu().numpy().astype(np.int64)
        for k in range(1, len(bad) - 1):
            lo, hi = bad[k - 1], min(bad[k - 1] + 1024, bad[k + 1])
            bad[k] = int(rng.integers(lo, hi + 1))
        try:
            E.decompress_chunked(t, E.RankIndex(1024, torch.from_numpy(bad).cuda()))
        except E.CorruptionError:
            pass
    # and the device is still healthy afterwards
    assert E.decompress_chunked(t, good).bytes() == w.tobytes()


@pytest.mark.parametrize("cs", [2048, 4096, 8192, 65536])
def test_chunked_coarse_index_fast_path(E, seeded_cases, cs):
    """decompress_chunked at the reference's default chunk size (4096,
    codec.hpp:19) and other coarse ones: count + per-entry index check + the TMA
    expand; bit-exact, and any wrong entry raises CorruptionError."""
    for i, c in enumerate(seeded_cases[:30]):
        rows, cols, eb = c["rows"], c["cols"], c["eb"]
        w = O.random_dense(rows, cols, eb, c["seed"], c["zero_fraction"])
        bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
        t = make_tensor(E, rows, cols, eb, bm, vals, nnz, values_offset=(i % 4) * eb)
        idx = E.build_rank_index(t.bitmap, cs)
        assert E.decompress_chunked(t, idx).bytes() == w.tobytes()
    rows, cols = 512, 1000
    w = O.random_dense(rows, cols, 2, 8, 0.5)
    bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
    t = make_tensor(E, rows, cols, 2, bm, vals, nnz)
    good = E.build_rank_index(t.bitmap, cs)
    assert E.decompress_chunked(t, good).bytes() == w.tobytes()
    if good.chunk_count() > 2:
        bad = good.prefix.clone()
        bad[1] += 1
        with pytest.raises(E.CorruptionError):
            E.decompress_chunked(t, E.RankIndex(cs, bad))


def test_chunks_any_order_and_isolation(E):
    # test_codec.cpp:168-200
    w = O.random_dense(16, 100, 1, 21, 0.5)
    bm, vals, nnz, _ = O.compress(w, 16, 100, 1)
    t = make_tensor(E, 16, 100, 1, bm, vals, nnz)
    idx = E.build_rank_index(t.bitmap, 128)
    assert idx.chunk_count() > 3
    buf = torch.zeros(t.dense_bytes(), dtype=torch.uint8, device="cuda")
    for k in reversed(range(idx.chunk_count())):
        E.decompress_chunk_into(t, idx, k, buf)
    assert buf.cpu().numpy().tobytes() == w.tobytes()

    w = O.random_dense(8, 64, 2, 5, 0.4)
    bm, vals, nnz, _ = O.compress(w, 8, 64, 2)
    t = make_tensor(E, 8, 64, 2, bm, vals, nnz)
    idx = E.build_rank_index(t.bitmap, 128)
    for k in range(idx.chunk_count()):
        buf = torch.full((t.dense_bytes(),), 0xAB, dtype=torch.uint8, device="cuda")
        E.decompress_chunk_into(t, idx, k, buf)
        got = buf.cpu().numpy()
        b, e = k * 128 * 2, min((k + 1) * 128 * 2, t.dense_bytes())
        assert (got[b:e] == w[b:e]).all()
        assert (got[:b] == 0xAB).all() and (got[e:] == 0xAB).all()


def test_large_chunk_into_spans_tiles(E):
    """cs larger than the 8192-element expand tile, and a ragged last chunk."""
    rows, cols = 301, 517
    w = O.random_dense(rows, cols, 2, 77, 0.45)
    bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
    t = make_tensor(E, rows, cols, 2, bm, vals, nnz)
    for cs in (16384, 65536):
        idx = E.build_rank_index(t.bitmap, cs)
        _, ref_p = O.rank_index(bm, rows * cols, cs)
        assert idx.prefix.cpu().numpy().astype(np.uint64).tolist() == ref_p.tolist()
        buf = torch.zeros(t.dense_bytes(), dtype=torch.uint8, device="cuda")
        for k in range(idx.chunk_count()):
            E.decompress_chunk_into(t, idx, k, buf)
        assert buf.cpu().numpy().tobytes() == w.tobytes()
        assert E.decompress_chunked(t, idx).bytes() == w.tobytes()


def test_index_errors(E):
    # test_codec.cpp:202-213: mismatched / truncated index -> CorruptionError
    w = O.random_dense(10, 10, 2, 9, 0.5)
    bm, vals, nnz, _ = O.compress(w, 10, 10, 2)
    t = make_tensor(E, 10, 10, 2, bm, vals, nnz)
    w2 = O.random_dense(10, 10, 2, 10, 0.2)
    bm2, _, _, _ = O.compress(w2, 10, 10, 2)
    bad = E.build_rank_index(E.Bitmap.from_bytes(bm2.tobytes(), 100, device="cuda"), 64)
    with pytest.raises(E.CorruptionError):
        E.decompress_chunked(t, bad)
    good = E.build_rank_index(t.bitmap, 64)
    trunc = E.RankIndex(64, good.prefix[:-1])
    with pytest.raises(E.CorruptionError):
        E.decompress_chunked(t, trunc)
    buf = torch.zeros(t.dense_bytes(), dtype=torch.uint8, device="cuda")
    with pytest.raises(E.BoundsError):
        E.decompress_chunk_into(t, good, good.chunk_count(), buf)
    with pytest.raises(E.InvalidArgument):
        E.decompress_chunk_into(t, good, 0, buf[:-2])
    with pytest.raises(E.CorruptionError):  # last prefix + tail != nnz
        E.decompress_chunk_into(t, bad, 0, buf)


# ---- acceptance.cpp criterion 3: 1000 cases ------------------------------------

def test_acceptance_1000(E, acceptance_cases):
    gold = {c["iter"]: c for c in acceptance_cases}
    for it, rows, cols, eb, zeros, w, chunk, _rsel, _csel in O.acceptance_cases(1000):
        g = gold[it]
        assert (rows, cols, eb, chunk) == (g["rows"], g["cols"], g["eb"], g["chunk"])
        assert crc(w) == g["crc_input"]
        dt = E.Dtype.F16 if eb == 2 else E.Dtype.I8
        t = E.compress(E.DenseMatrix.from_host(rows, cols, dt, w.tobytes()))
        assert t.nnz() == g["nnz"], it
        assert crc(t.bitmap.data) == g["crc_bitmap"] and crc(t.values) == g["crc_values"], it
        full = E.decompress(t)
        assert crc(full.data) == g["crc_dense"], it
        idx = E.build_rank_index(t.bitmap, chunk)
        assert crc(idx.prefix.cpu().numpy().astype("<u8")) == g["crc_prefix"], it
        assert crc(E.decompress_chunked(t, idx).data) == g["crc_dense"], it


# ---- GEMV consumer (fp32 reference, 1e-3 relative) --------------------------------

@pytest.mark.parametrize("rows,cols", [(1, 8), (33, 64), (257, 1000), (1024, 9216), (130, 36864)])
def test_gemv_matches_fp32_reference(E, rows, cols):
    g = torch.Generator(device="cpu").manual_seed(rows * 7 + cols)
    W = (torch.rand(rows, cols, generator=g) * 2 - 1).half()
    x = (torch.rand(cols, generator=g) * 2 - 1).half()
    ref = W.float() @ x.float()
    Wd = E.DenseMatrix.from_host(rows, cols, E.Dtype.F16, W.view(torch.uint8).reshape(-1))
    y = E.gemv(Wd, x.cuda()).cpu()
    from conftest import gemv_check
    gemv_check(y, W, x)


def test_concurrent_host_threads_disjoint_chunks(E):
    """SPEC.md:143-144 / codec.hpp:188-190: per-chunk calls into disjoint regions
    may run concurrently.  Four host threads, each with its own stream and
    workspace, decompress_chunk_into interleaved chunks of one tensor into one
    buffer; the result is the reference's decompress."""
    import threading
    rows, cols = 257, 1031
    w = O.random_dense(rows, cols, 2, 606, 0.45)
    bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
    t = make_tensor(E, rows, cols, 2, bm, vals, nnz)
    idx = E.build_rank_index(t.bitmap, 4096)
    buf = torch.zeros(t.dense_bytes(), dtype=torch.uint8, device="cuda")
    errs = []

    def worker(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for k in range(r, idx.chunk_count(), 4):
                    E.decompress_chunk_into(t, idx, k, buf)
            s.synchronize()
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    torch.cuda.synchronize()
    assert not errs
    assert buf.cpu().numpy().tobytes() == w.tobytes()


def _host_prefix(bm, n, cs):
    """RankIndex(cs, prefix) for ANY nonzero chunk size (the reference's
    RankIndex constructor accepts it, bitmap.hpp:104; check_index and
    scatter_range work with it, codec.hpp:132-216)."""
    bits = np.unpackbits(np.asarray(bm, dtype=np.uint8), bitorder="little")[:n].astype(np.int64)
    cum = np.concatenate([[0], np.cumsum(bits)])
    return cum[np.arange(0, n, cs)]


@pytest.mark.parametrize("cs", [1, 3, 31, 100, 1000, 1500, 2048, 4095, 5000, 9999])
@pytest.mark.parametrize("eb", [1, 2])
def test_arbitrary_chunk_sizes(E, cs, eb):
    """decompress_chunked / decompress_chunk_into at chunk sizes that are not
    powers of two (chunk ranges start and end inside bitmap words): output
    == the reference's, every chunk writes exactly its own range (0xAB
    sentinel, test_codec.cpp:181-200), a corrupted middle entry is rejected."""
    rows, cols = 37, 613 if cs > 64 else 41
    w = O.random_dense(rows, cols, eb, 900 + cs, 0.45)
    bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
    t = make_tensor(E, rows, cols, eb, bm, vals, nnz)
    n = rows * cols
    pre = _host_prefix(bm, n, cs)
    idx = E.RankIndex(cs, torch.from_numpy(pre).cuda())
    assert E.decompress_chunked(t, idx).bytes() == w.tobytes()
    # unaligned bitmap (plain scan + expand path)
    ub = torch.zeros(len(bm) + 20, dtype=torch.uint8, device="cuda")[4:4 + len(bm)]
    ub.copy_(torch.from_numpy(bm.copy()))
    tu = E.EndorTensor(rows, cols, t.dtype, E.Bitmap(n, data=ub), t.values, validate=False, nnz=nnz)
    assert E.decompress_chunked(tu, idx).bytes() == w.tobytes()
    ks = list(range(idx.chunk_count()))
    for k in (ks if len(ks) <= 24 else ks[:8] + ks[len(ks) // 2: len(ks) // 2 + 4] + ks[-8:]):
        buf = torch.full((t.dense_bytes(),), 0xAB, dtype=torch.uint8, device="cuda")
        E.decompress_chunk_into(t, idx, k, buf)
        got = buf.cpu().numpy()
        b, e = k * cs * eb, min((k + 1) * cs, n) * eb
        assert (got[b:e] == w[b:e]).all(), k
        assert (got[:b] == 0xAB).all() and (got[e:] == 0xAB).all(), k
    full = torch.zeros(t.dense_bytes(), dtype=torch.uint8, device="cuda")
    for k in reversed(ks):
        E.decompress_chunk_into(t, idx, k, full)
    assert full.cpu().numpy().tobytes() == w.tobytes()
    if len(pre) > 2:
        bad = pre.copy()
        bad[len(pre) // 2] += 1
        with pytest.raises(E.CorruptionError):
            E.decompress_chunked(t, E.RankIndex(cs, torch.from_numpy(bad).cuda()))
        bad_last = pre.copy()
        bad_last[-1] += 1
        with pytest.raises(E.CorruptionError):
            E.decompress_chunk_into(t, E.RankIndex(cs, torch.from_numpy(bad_last).cuda()), 0, full)


def test_empty_tensor_chunk_into_host_bounds(E):
    """an empty tensor through the host-buffer chunk_into must raise
    BoundsError (check_index passes with 0 chunks, codec.hpp:172-177,194), not
    read before the prefix allocation."""
    import ctypes as C
    L = E._lib.lib()
    dst = (C.c_uint8 * 1)()
    st = L.endor_cuda_decompress_chunk_into_host(0, 5, 0, None, None, 0, 64, None, 0, 0, dst, 0)
    assert st == 3, L.endor_cuda_last_error_string()  # ENDOR_ERR_BOUNDS
    st = L.endor_cuda_decompress_chunk_into_host(4, 0, 1, None, None, 0, 4096, None, 0, 2, dst, 0)
    assert st == 3
