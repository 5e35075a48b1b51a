"""Uneven per-tile density (GPU): every TMA window size from
empty to a fully dense 16 KiB item, and structured sparsity.

Patterns on a 96 x 16384 f16 matrix (192 expand tiles, 1536 RankIndex chunks):
N:M pruning (2:4, 1:4, 3:4 via the reference's nm_prune restated in the
oracle, weight_gen.hpp:118-141), alternating fully dense / empty rows,
half-dense rows, alternating dense / empty 8192-element tiles, a per-row
density ramp 0 -> 100 %, and a single set element.  Each is checked
bit-exact for decompress (count + TMA expand), decompress_chunked at chunk
1024 (single launch) and 4096 (coarse index), extract_rows / extract_cols,
and the fused decompress -> GEMV against an fp32 GEMV over the dense matrix
(north star tolerance 1e-3 relative, element-wise: conftest.gemv_check).
"""
import numpy as np
import pytest

from conftest import gemv_check  # noqa: E402

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

ROWS, COLS = 96, 16384


def _values(rng, n):
    # finite non-zero f16 bit patterns in [-1, 1): never +-0, so the mask decides
    mag = rng.integers(0x0400, 0x3C00, n, dtype=np.uint16)
    sign = rng.integers(0, 2, n, dtype=np.uint16) << 15
    return (mag | sign).astype(np.uint16)


def _patterns():
    rng = np.random.default_rng(11)
    n = ROWS * COLS
    ramp = np.zeros((ROWS, COLS), bool)
    for r in range(ROWS):
        ramp[r] = rng.random(COLS) < r / (ROWS - 1)
    tiles = (np.arange(n) // 8192 % 2 == 0).reshape(ROWS, COLS)
    one = np.zeros((ROWS, COLS), bool)
    one[ROWS // 2, COLS // 3] = True
    masks = {
        "rows_dense_empty": np.repeat((np.arange(ROWS) % 2 == 0)[:, None], COLS, 1),
        "half_rows": np.repeat((np.arange(COLS) < COLS // 2)[None, :], ROWS, 0),
        "tiles_dense_empty": tiles,
        "density_ramp": ramp,
        "single": one,
        "all_dense": np.ones((ROWS, COLS), bool),
    }
    for name, m in masks.items():
        yield name, np.where(m, _values(rng, n).reshape(ROWS, COLS), 0).astype(np.uint16)
    for keep, m in ((2, 4), (1, 4), (3, 4)):
        w = _values(rng, n).view(np.uint8).copy()
        out = np.zeros_like(w)
        assert O.lib().or_nm_prune(ROWS, COLS, 2, keep, m, w, out) == 0
        yield f"nm{keep}:{m}", out.view(np.uint16).reshape(ROWS, COLS)


@pytest.mark.parametrize("name,w", list(_patterns()), ids=lambda v: v if isinstance(v, str) else "")
def test_density_pattern(cuda_lib, name, w):
    from paper_2406_11674_b200 import codec as E
    raw = np.ascontiguousarray(w).view(np.uint8).reshape(-1)
    bm, vals, nnz, _ = O.compress(raw, ROWS, COLS, 2)
    b = torch.zeros(len(bm) + 32, dtype=torch.uint8, device="cuda")[: len(bm)]
    b.copy_(torch.from_numpy(bm))
    v = torch.zeros(len(vals) + 64, dtype=torch.uint8, device="cuda")[1: 1 + len(vals)]  # odd value offset
    if len(vals):
        v.copy_(torch.from_numpy(vals))
    t = E.EndorTensor(ROWS, COLS, E.Dtype.F16, E.Bitmap(ROWS * COLS, data=b), v, validate=False, nnz=nnz)
    want = raw.tobytes()
    assert E.decompress(t).bytes() == want, name
    for cs in (1024, 4096):
        assert E.decompress_chunked(t, E.build_rank_index(t.bitmap, cs)).bytes() == want, (name, cs)
    full = raw.reshape(ROWS, COLS * 2)
    rsel = [0, 1, ROWS // 2, ROWS - 1]
    assert E.extract_rows(t, rsel).bytes() == full[rsel].tobytes(), name
    csel = sorted({0, 1, 8191, 8192, COLS // 3, COLS - 1} | set(range(100, COLS, 97)))
    assert E.extract_cols(t, csel).bytes() == np.ascontiguousarray(w[:, csel]).tobytes(), name
    x = (torch.rand(COLS, device="cuda", generator=torch.Generator("cuda").manual_seed(2)) * 2 - 1).half()
    y = E.gemv_compressed(t, x)
    gemv_check(y, torch.from_numpy(np.ascontiguousarray(w).view(np.float16)), x)
