"""decompress_chunked with a coarse RankIndex (chunk 2048 / 4096 / 8192 -- the
reference's default is kDefaultChunkSize = 4096, codec.hpp:19) in ONE expand
launch: the producer derives each 1024-element sub-tile's start from the
chunk entries and the staged bitmap, and checks every entry (check_index,
codec.hpp:170-184, plus the middle entries the multi-launch path also checks).

Bit-exact against the oracle on ragged shapes, both dtypes and unaligned
value buffers; every wrong entry -- first, middle, last, shifted suffixes,
adversarial values -- raises CorruptionError and leaves the device healthy.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E(cuda_lib):
    from paper_2406_11674_b200 import codec
    return codec


def dev_bytes(a, offset=0):
    a = np.ascontiguousarray(np.asarray(a).view(np.uint8).reshape(-1))
    buf = torch.zeros(a.size + offset + 32, dtype=torch.uint8, device="cuda")
    view = buf[offset: offset + a.size]
    if a.size:
        view.copy_(torch.from_numpy(a.copy()))
    return view


def tensor(E, rows, cols, eb, seed, zero_fraction, values_offset=0):
    w = O.random_dense(rows, cols, eb, seed, zero_fraction)
    bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
    n = rows * cols
    dt = E.Dtype.F16 if eb == 2 else E.Dtype.I8
    t = E.EndorTensor(rows, cols, dt, E.Bitmap(n, data=dev_bytes(bm)), dev_bytes(vals, values_offset),
                      validate=False, nnz=nnz)
    return w, bm, t


SHAPES = [(1, 1), (1, 8191), (1, 8193), (3, 8197), (64, 8192), (17, 12345), (1000, 333), (2, 4096), (5, 2049)]


@pytest.mark.parametrize("cs", [2048, 4096, 8192])
@pytest.mark.parametrize("eb", [1, 2])
def test_coarse_index_bit_exact(E, cs, eb):
    for i, (rows, cols) in enumerate(SHAPES):
        for zf in (0.0, 0.5, 0.93, 1.0):
            w, bm, t = tensor(E, rows, cols, eb, 100 * i + int(zf * 10) + cs, zf, values_offset=(i % 4) * eb)
            idx = E.build_rank_index(t.bitmap, cs)
            _, pre = O.rank_index(bm, rows * cols, cs)
            assert idx.prefix.cpu().numpy().astype(np.uint64).tolist() == pre.tolist()
            assert E.decompress_chunked(t, idx).bytes() == w.tobytes(), (rows, cols, zf)


@pytest.mark.parametrize("cs", [2048, 4096, 8192])
def test_every_wrong_entry_is_rejected(E, cs):
    rows, cols = 40, 3000  # 120000 elements: 59 / 30 / 15 chunks, ragged last tile
    w, bm, t = tensor(E, rows, cols, 2, 77 + cs, 0.5)
    good = E.build_rank_index(t.bitmap, cs)
    nch = good.chunk_count()
    pre = good.prefix.cpu().numpy().astype(np.int64)
    positions = sorted({0, 1, 2, nch // 2, nch - 2, nch - 1})
    for k in positions:
        for d in (+1, -1, +7):
            bad = pre.copy()
            bad[k] += d
            if bad[k] < 0:
                continue
            with pytest.raises(E.CorruptionError):
                E.decompress_chunked(t, E.RankIndex(cs, torch.from_numpy(bad).cuda()))
        # every entry from k on shifted by one: only the first shifted chunk boundary disagrees
        bad = pre.copy()
        bad[k:] += 1
        with pytest.raises(E.CorruptionError):
            E.decompress_chunked(t, E.RankIndex(cs, torch.from_numpy(bad).cuda()))
    for v in (10 ** 12, -5, 2 ** 40):  # out-of-range values: clamped in the producer, reported
        bad = pre.copy()
        bad[nch // 2] = v
        with pytest.raises(E.CorruptionError):
            E.decompress_chunked(t, E.RankIndex(cs, torch.from_numpy(bad).cuda()))
    rng = np.random.default_rng(cs)
    for _ in range(10):  # random monotone garbage with the right last entry
        bad = np.sort(rng.integers(0, int(t.nnz()) + 1, size=nch)).astype(np.int64)
        bad[0] = 0
        bad[-1] = pre[-1]
        if (bad == pre).all():
            continue
        with pytest.raises(E.CorruptionError):
            E.decompress_chunked(t, E.RankIndex(cs, torch.from_numpy(bad).cuda()))
    assert E.decompress_chunked(t, good).bytes() == w.tobytes()  # device healthy


@pytest.mark.parametrize("eb", [1, 2])
def test_coarse_index_batch(E, eb):
    """decompress_batch with 4096-chunk indices: one launch for the batch."""
    shapes = [(9, 8192), (33, 1000), (1, 5), (128, 513)]
    ws, ts = [], []
    for i, (r, c) in enumerate(shapes):
        w, _, t = tensor(E, r, c, eb, 500 + i, 0.4, values_offset=i % 3 * eb)
        ws.append(w)
        ts.append(t)
    outs = E.decompress_batch(ts, indices=[E.build_rank_index(t.bitmap, 4096) for t in ts])
    for w, o in zip(ws, outs):
        assert o.bytes() == w.tobytes()


def test_coarse_index_layer_shape(E):
    """One OPT-66B fc1 (9216 x 36864 @ 50 %) through the 4096-chunk index."""
    w = E.synth_weight(9216, 36864, 7, device="cuda")
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    for cs in (2048, 4096, 8192):
        assert torch.equal(E.decompress_chunked(t, E.build_rank_index(t.bitmap, cs)).data, w.data), cs


def test_pool_claims_recover_after_latched_error(E):
    """A layer-sized launch takes its last tiles from the shared pool counter
    in the workspace (expand.cu, ENDOR_TMA_GLOBAL_CLAIMS); CTAs that see a
    latched error skip that protocol, so the status reset must also reset the
    counter -- every later launch on the same (cached) workspace is bit-exact."""
    w = E.synth_weight(8192, 32768, 11, device="cuda")
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    for cs in (1024, 4096):
        good = E.build_rank_index(t.bitmap, cs)
        pre = good.prefix.cpu().numpy().astype(np.int64)
        for k in (1, len(pre) // 3, len(pre) - 2):
            bad = pre.copy()
            bad[k:] += 3
            with pytest.raises(E.CorruptionError):
                E.decompress_chunked(t, E.RankIndex(cs, torch.from_numpy(bad).cuda()))
            for _ in range(3):
                assert torch.equal(E.decompress_chunked(t, good).data, w.data), (cs, k)
            assert torch.equal(E.decompress(t).data, w.data), (cs, k)
