"""Tensors past 2^32 elements (GPU): every 64-bit offset path.

The reference counts elements and bytes in u64 (`dense_matrix.hpp:28-33`,
`checked_element_count`); real embedding / LM-head matrices exceed 4 GiB of
dense bytes (128256 x 16384 f16 = 4.2 GB).  These cases cross the 2^32
element boundary (65537 x 65536 = 4,295,032,832 elements, 8.6 GB dense f16)
and check, on the device chain synth -> prune -> compress:

* decompress / decompress_chunked (chunk 1024 and 4096) round-trip to W;
* rows on both sides of element 2^32 against a numpy expansion of the
  bitmap + values bytes (rank from a RankIndex at chunk = cols);
* decompress_chunk_into of the last chunk (a partial range past 2^32);
* extract_rows of the last rows, the fused GEMV against the dense GEMV;
* the same round trip for i8 (4.3 GB dense).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROWS, COLS = 65537, 65536  # row 65536 starts exactly at element 2^32


def _row_from_bytes(t, idx_rows, r):
    """numpy expansion of row r from the compressed bytes (bitmap.hpp:14-17 bit order)."""
    eb = 2 if int(t.dtype) == 0 else 1
    c = t.cols
    bm = t.bitmap.data[r * c // 8:(r + 1) * c // 8].cpu().numpy()
    bits = np.unpackbits(bm, bitorder="little").astype(bool)
    v0 = int(idx_rows.prefix[r].item())
    k = int(bits.sum())
    vals = t.values[v0 * eb:(v0 + k) * eb].cpu().numpy()
    dense = np.zeros(c * eb, dtype=np.uint8).reshape(c, eb)
    dense[bits] = vals.reshape(k, eb)
    return dense.reshape(-1)


def test_f16_past_2p32(cuda_lib):
    from paper_2406_11674_b200 import codec as E
    n = ROWS * COLS
    assert n > 1 << 32
    w = E.synth_weight(ROWS, COLS, 11, device="cuda")
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    assert t.nnz() == n - int(0.5 * n)
    wb = w.data.view(torch.uint8).reshape(ROWS, COLS * 2)

    out = E.decompress(t)                                     # count + TMA expand
    assert torch.equal(out.data, w.data)
    del out
    idx_rows = E.build_rank_index(t.bitmap, COLS)             # one entry per row
    for r in (0, ROWS // 2, ROWS - 2, ROWS - 1):
        got = wb[r].cpu().numpy()
        assert np.array_equal(got, _row_from_bytes(t, idx_rows, r)), r

    for cs in (1024, 4096):
        idx = E.build_rank_index(t.bitmap, cs)
        out = E.decompress_chunked(t, idx)
        assert torch.equal(out.data, w.data), cs
        del out
    # a partial range past 2^32: the last chunk only, into a zeroed full buffer
    idx = E.build_rank_index(t.bitmap, 1 << 20)
    dst = torch.zeros(n * 2, dtype=torch.uint8, device="cuda")
    k = idx.chunk_count() - 1
    E.decompress_chunk_into(t, idx, k, dst)
    lo = k * (1 << 20) * 2
    assert torch.equal(dst[lo:], w.data.view(torch.uint8).reshape(-1)[lo:])
    assert int(dst[:lo].count_nonzero().item()) == 0
    del dst

    sel = [ROWS // 3, ROWS - 2, ROWS - 1]
    assert torch.equal(E.extract_rows(t, sel).data.view(torch.uint8).reshape(len(sel), -1), wb[sel])

    x = (torch.rand(COLS, device="cuda", generator=torch.Generator("cuda").manual_seed(3)) * 2 - 1).half()
    y = E.gemv_compressed(t, x)
    ref = E.gemv(w, x)  # the dense kernel over the same W: agree within fp32 rounding, per row
    wabs = E.DenseMatrix(ROWS, COLS, E.Dtype.F16, w.data.view(torch.float16).abs().view(torch.uint8))
    mag = E.gemv(wabs, x.abs())  # sum_j |W_ij x_j| (the row's conditioning), element-wise bound
    assert ((y - ref).abs() <= 1e-3 * mag).all()
    good = ref.abs() >= 0.01 * mag
    assert ((y - ref)[good].abs() <= 1e-3 * ref[good].abs()).all()
    del wabs, mag
    del w, t, wb
    torch.cuda.empty_cache()


def test_i8_past_2p32(cuda_lib):
    from paper_2406_11674_b200 import codec as E
    w = E.synth_weight(ROWS, COLS, 12, dtype=E.Dtype.I8, device="cuda")
    E.magnitude_prune(w, 0.6, inplace=True)
    t = E.compress(w)
    out = E.decompress(t)
    assert torch.equal(out.data, w.data)
    idx_rows = E.build_rank_index(t.bitmap, COLS)
    wb = w.data.view(torch.uint8).reshape(ROWS, COLS)
    for r in (ROWS - 2, ROWS - 1):
        assert np.array_equal(wb[r].cpu().numpy(), _row_from_bytes(t, idx_rows, r)), r
    idx = E.build_rank_index(t.bitmap, 1024)
    assert torch.equal(E.decompress_chunked(t, idx).data, w.data)
    del w, t, out
    torch.cuda.empty_cache()
