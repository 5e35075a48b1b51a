"""§8(f) row 4: selective row/column decompression on the GPU against the
reference's semantics: extraction == slicing the full decompression
(acceptance.cpp:126-153), index validation as check_sorted_unique
(codec.hpp:224-232)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E(cuda_lib):
    from paper_2406_11674_b200 import codec
    return codec


def _tensor(E, rows, cols, eb, bm, vals, nnz, voff=0):
    n = rows * cols
    b = torch.zeros(len(bm) + 32, dtype=torch.uint8, device="cuda")[: len(bm)]
    if len(bm):
        b.copy_(torch.from_numpy(bm.copy()))
    v = torch.zeros(len(vals) + voff + 32, dtype=torch.uint8, device="cuda")[voff: voff + len(vals)]
    if len(vals):
        v.copy_(torch.from_numpy(vals.copy()))
    dt = E.Dtype.F16 if eb == 2 else E.Dtype.I8
    return E.EndorTensor(rows, cols, dt, E.Bitmap(n, data=b), v, validate=False, nnz=nnz)


def test_acceptance_extraction_suite(E):
    """acceptance.cpp criterion 3's extraction half, 1000 generated cases."""
    for it, rows, cols, eb, zeros, w, chunk, rsel, csel in O.acceptance_cases(1000):
        if it % 4:  # a quarter of the suite keeps the GPU run short; all shapes classes included
            continue
        bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
        t = _tensor(E, rows, cols, eb, bm, vals, nnz, voff=it % 3)
        full = w.reshape(rows, cols * eb)
        gr = E.extract_rows(t, rsel)
        assert gr.bytes() == full[rsel].tobytes() if rsel else gr.bytes() == b"", it
        gc = E.extract_cols(t, csel)
        want = w.view(np.uint16 if eb == 2 else np.uint8).reshape(rows, cols)[:, csel]
        assert gc.bytes() == np.ascontiguousarray(want).tobytes(), it


def test_large_rows_and_cols(E):
    rows, cols = 9216, 36864
    w = E.synth_weight(rows, cols, 7, device="cuda")
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    dense = w.data.view(torch.int16).reshape(rows, cols)
    rsel = torch.arange(3, rows, 97, device="cuda")
    got = E.extract_rows(t, rsel)
    assert torch.equal(got.data.view(torch.int16).reshape(-1, cols), dense[rsel])
    for step in (131, 2, 1):  # direct lookups (sparse selection), tiled (half, all columns)
        csel = torch.arange(5 % step, cols, step, device="cuda")
        got = E.extract_cols(t, csel)
        assert torch.equal(got.data.view(torch.int16).reshape(rows, -1), dense[:, csel]), step


def test_extract_rows_expand_ring_shapes(E):
    """extract_rows with cols % 1024 == 0 (the TMA expand ring over (row, tile)
    items): odd 1024-chunk row starts (unaligned index entries), partial last
    tiles, both dtypes, any value-buffer alignment, first / last / all rows."""
    for rows, cols, eb, zf, voff in ((7, 3072, 2, 0.5, 1), (5, 9216, 2, 0.3, 0), (33, 1024, 1, 0.6, 3),
                                     (4, 16384, 2, 0.9, 2), (3, 8192, 1, 0.0, 0), (2, 2048, 2, 1.0, 0)):
        w = O.random_dense(rows, cols, eb, rows * 7 + cols, zf)
        bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
        t = _tensor(E, rows, cols, eb, bm, vals, nnz, voff=voff)
        full = w.reshape(rows, cols * eb)
        for rsel in ([0], [rows - 1], list(range(rows)), list(range(1, rows, 2)), [0, rows - 1]):
            rsel = sorted(set(rsel))
            assert E.extract_rows(t, rsel).bytes() == full[rsel].tobytes(), (rows, cols, eb, rsel)


@pytest.mark.parametrize("rpc", [1, 3])
def test_extract_cols_rows_per_cta(cuda_lib, rpc):
    """extract_cols with 1 and 3 rows per CTA (the default is 4) over the
    acceptance subset and ragged shapes, each in a fresh process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, torch\n"
        "from oracle import oracle as O\n"
        "from paper_2406_11674_b200 import codec as E\n"
        "for it, rows, cols, eb, zeros, w, chunk, rsel, csel in O.acceptance_cases(300):\n"
        "    bm, vals, nnz, _ = O.compress(w, rows, cols, eb)\n"
        "    b = torch.zeros(len(bm) + 32, dtype=torch.uint8, device='cuda')[:len(bm)]\n"
        "    b.copy_(torch.from_numpy(bm.copy())) if len(bm) else None\n"
        "    off = it % 3\n"
        "    v = torch.zeros(len(vals) + off + 32, dtype=torch.uint8, device='cuda')[off:off + len(vals)]\n"
        "    v.copy_(torch.from_numpy(vals.copy())) if len(vals) else None\n"
        "    t = E.EndorTensor(rows, cols, E.Dtype.F16 if eb == 2 else E.Dtype.I8, E.Bitmap(rows * cols, data=b), v,\n"
        "                      validate=False, nnz=nnz)\n"
        "    want = w.view(np.uint16 if eb == 2 else np.uint8).reshape(rows, cols)[:, csel]\n"
        "    assert E.extract_cols(t, csel).bytes() == np.ascontiguousarray(want).tobytes(), it\n"
        "for rows, cols, eb in ((3, 20000, 2), (70, 8193, 1), (5, 16384, 2), (37, 3072, 2), (1, 1024, 2), (9, 8, 2), (300, 40, 2), (2, 8200, 2)):\n"
        "    w = O.random_dense(rows, cols, eb, rows + cols, 0.5)\n"
        "    bm, vals, nnz, _ = O.compress(w, rows, cols, eb)\n"
        "    t = E.EndorTensor(rows, cols, E.Dtype.F16 if eb == 2 else E.Dtype.I8,\n"
        "                      E.Bitmap(rows * cols, data=torch.from_numpy(bm.copy()).cuda()),\n"
        "                      torch.from_numpy(vals.copy()).cuda(), validate=False, nnz=nnz)\n"
        "    for csel in ([0], [cols - 1], list(range(0, cols, 7)), [8191, 8192, cols - 1], list(range(cols)),\n"
        "                 list(range(1000, cols, 2)), list(range(cols - 40, cols))):\n"
        "        csel = sorted({c for c in csel if 0 <= c < cols})\n"
        "        want = w.view(np.uint16 if eb == 2 else np.uint8).reshape(rows, cols)[:, csel]\n"
        "        assert E.extract_cols(t, csel).bytes() == np.ascontiguousarray(want).tobytes(), (rows, cols, csel[:3])\n"
        "print('ok')\n")
    env = dict(os.environ, ENDOR_EXTRACT_COLS_RPC=str(rpc), PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]


def test_index_validation_matches_reference(E):
    w = O.random_dense(10, 12, 2, 9, 0.5)
    bm, vals, nnz, _ = O.compress(w, 10, 12, 2)
    t = _tensor(E, 10, 12, 2, bm, vals, nnz)
    R = O.ref()
    cases = [([1, 10], "rows", E.BoundsError), ([3, 3], "rows", E.InvalidArgument),
             ([4, 2], "rows", E.InvalidArgument), ([2, 1, 99], "rows", E.InvalidArgument),
             ([99, 1], "rows", E.BoundsError), ([0, 12], "cols", E.BoundsError),
             ([5, 5, 99], "cols", E.InvalidArgument)]
    for sel, kind, exc in cases:
        with pytest.raises(exc):
            (E.extract_rows if kind == "rows" else E.extract_cols)(t, sel)
        if R is not None:
            out = np.zeros(4096, np.uint8)
            code = R.ref_extract(10, 12, 2, bm, vals, nnz, np.array(sel, np.uint64), len(sel),
                                 1 if kind == "rows" else 0, out)
            assert code == (3 if exc is E.BoundsError else 4)
    # empty selections are valid
    assert E.extract_rows(t, []).bytes() == b""
    assert E.extract_cols(t, []).bytes() == b""
