"""§8(f) row 1: fused decompress -> GEMV (y = W x from the compressed W).
Floating point: checked against an fp32 reference GEMV over the reference-
exact decompressed W, max|y - y_ref| <= 1e-3 * max|y_ref| (north star's 1e-3
relative tolerance), and bit-identical across runs (deterministic order)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E(cuda_lib):
    from paper_2406_11674_b200 import codec
    return codec


@pytest.mark.parametrize("rows,cols,s", [(1, 1024, 0.5), (37, 2048, 0.0), (300, 9216, 0.5), (64, 36864, 0.9),
                                         (1024, 8192, 0.3)])
def test_fused_gemv_matches_fp32_reference(E, rows, cols, s):
    w = E.synth_weight(rows, cols, rows * 31 + cols, device="cuda")
    if s > 0:
        E.magnitude_prune(w, s, inplace=True)
    t = E.compress(w)
    g = torch.Generator(device="cpu").manual_seed(cols)
    x = ((torch.rand(cols, generator=g) * 2 - 1).half()).cuda()
    Wd = w.data.view(torch.float16).reshape(rows, cols).float()
    ref = Wd @ x.float()
    tol = 1e-3 * ref.abs().max().item() + 1e-6
    y = E.gemv_compressed(t, x)
    assert (y - ref).abs().max().item() <= tol
    y2 = E.gemv_compressed(t, x, index=E.build_rank_index(t.bitmap, 1024))
    assert torch.equal(y, y2)              # same partials, same order
    assert torch.equal(y, E.gemv_compressed(t, x))  # deterministic
    # and equal to the materialised path within fp32 rounding
    yd = E.gemv(E.decompress(t), x)
    assert (y - yd).abs().max().item() <= tol


def test_fused_gemv_rejects_unsupported(E):
    w = O.random_dense(4, 1000, 2, 1, 0.5)
    bm, vals, nnz, _ = O.compress(w, 4, 1000, 2)
    b = torch.zeros(len(bm) + 32, dtype=torch.uint8, device="cuda")[: len(bm)]
    b.copy_(torch.from_numpy(bm))
    v = torch.from_numpy(vals.copy()).cuda()
    t = E.EndorTensor(4, 1000, E.Dtype.F16, E.Bitmap(4000, data=b), v)
    with pytest.raises(E.InvalidArgument):  # cols % 1024 != 0
        E.gemv_compressed(t, torch.zeros(1000, dtype=torch.float16, device="cuda"))
