"""North star (b) "dense GEMV/GEMM consumer", the GEMM half: Y = X W^T from
the compressed W by the fused decompress -> tcgen05 GEMM
(csrc/gemm_fused.cu; the reference models this consumer only as a constant,
sim.hpp:30,256).  Floating point: checked element-wise against a float64
product over the reference-exact W (conftest.gemm_check: 1e-3 of sum|X W| per
entry, 1e-3 relative where not cancellation-dominated), bit-identical across
runs and with / without a caller RankIndex; W itself comes from the
reference-exact synth_weight + magnitude_prune + compress chain (bit-exact vs
the oracle, test_gpu_parity.py), and the oracle's own compress feeds the
ragged cases."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import gemm_check  # noqa: E402
from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E(cuda_lib):
    from paper_2406_11674_b200 import codec
    return codec


def _x(tokens, cols, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return ((torch.rand(tokens, cols, generator=g) * 2 - 1).half()).cuda()


def _synth(E, rows, cols, s, seed):
    w = E.synth_weight(rows, cols, seed, device="cuda")
    if s > 0:
        E.magnitude_prune(w, s, inplace=True)
    return E.compress(w), w.data.view(torch.float16).reshape(rows, cols)


def _oracle_tensor(E, rows, cols, s, seed, values_offset=0):
    """ragged shapes straight from the oracle's compress; values_offset > 0
    places the packed values at an odd 2-byte offset (exercises the bytewise
    window path at the buffer ends)"""
    w = O.random_dense(rows, cols, 2, seed, s)
    bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
    b = torch.from_numpy(bm.copy()).cuda()
    vb = torch.zeros(len(vals) + 64, dtype=torch.uint8, device="cuda")
    v = vb[values_offset:values_offset + len(vals)]
    v.copy_(torch.from_numpy(vals.copy()))
    t = E.EndorTensor(rows, cols, E.Dtype.F16, E.Bitmap(rows * cols, data=b), v)
    W = torch.from_numpy(w.view(np.uint16).astype(np.int32)).to(torch.int16).view(torch.float16).reshape(rows, cols)
    return t, W


@pytest.mark.parametrize("rows,cols,tokens,s", [
    (128, 128, 16, 0.5),      # one tile, one span
    (128, 1024, 64, 0.0),     # dense W
    (256, 2048, 1, 0.5),      # decode batch of one
    (300, 1024, 100, 0.7),    # ragged rows, BN = 128
    (129, 4096, 256, 0.5),    # BN = 256, one row in the second m-tile
    (384, 2048, 300, 0.9),    # two n-tiles, the second mostly padding
    (512, 9216, 33, 0.5),     # OPT-66B attention width, split-K
    (64, 36864, 8, 0.5),      # fc2 width: deep K, many splits
])
def test_gemm_matches_fp64_reference(E, rows, cols, tokens, s):
    t, W = _synth(E, rows, cols, s, rows * 7 + cols + tokens)
    X = _x(tokens, cols, cols + tokens)
    y = E.gemm_compressed(t, X)
    gemm_check(y, W, X)
    y2 = E.gemm_compressed(t, X, index=E.build_rank_index(t.bitmap, 1024))
    assert torch.equal(y, y2)             # same tiles, same order
    assert torch.equal(y, E.gemm_compressed(t, X))  # deterministic
    yh = E.gemm_compressed(t, X, out_dtype=torch.float16)
    assert torch.equal(yh, y.half())      # f16 output = RNE of the fp32 result


@pytest.mark.parametrize("rows,cols,tokens,s,off", [
    (96, 1000, 5, 0.5, 0),    # cols % 128 != 0: generic bitmap path, X rows padded
    (33, 77, 3, 0.3, 2),      # tiny, unaligned values pointer
    (130, 200, 70, 0.6, 6),   # ragged everything
    (7, 129, 17, 0.0, 2),     # dense, one column past a span
    (5, 64, 2, 1.0, 0),       # all pruned: Y = 0
])
def test_gemm_ragged_shapes(E, rows, cols, tokens, s, off):
    t, W = _oracle_tensor(E, rows, cols, s, rows + cols, values_offset=off)
    X = _x(tokens, cols, rows * cols)
    y = E.gemm_compressed(t, X)
    gemm_check(y, W, X)
    if s >= 1.0:
        assert not y.any()


def test_gemm_equals_gemv_per_token(E):
    rows, cols = 256, 9216
    t, W = _synth(E, rows, cols, 0.5, 11)
    X = _x(4, cols, 5)
    y = E.gemm_compressed(t, X)
    for i in range(4):
        yv = E.gemv_compressed(t, X[i].contiguous())
        torch.testing.assert_close(y[i], yv, rtol=2e-5, atol=1e-4)


def test_gemm_errors_latched(E):
    rows, cols = 256, 1024
    t, _ = _synth(E, rows, cols, 0.5, 3)
    X = _x(16, cols, 1)
    # values length disagrees with the bitmap popcount (codec.hpp:158-160)
    bad = E.EndorTensor(rows, cols, E.Dtype.F16, t.bitmap, t.values[:-2], validate=False)
    with pytest.raises(E.CorruptionError):
        E.gemm_compressed(bad, X)
    # an inconsistent caller index
    idx = E.build_rank_index(t.bitmap, 1024)
    p = idx.prefix.clone()
    p[3] += 5
    idx2 = E.RankIndex(1024, p)
    with pytest.raises(E.CorruptionError):
        E.gemm_compressed(t, X, index=idx2)
    # the workspace stays usable after a latched error
    gemm_check(E.gemm_compressed(t, X), t_dense(E, t), X)


def t_dense(E, t):
    return E.decompress(t).data.view(torch.float16).reshape(t.rows, t.cols)


def test_gemm_rejects_bad_args(E):
    t, _ = _synth(E, 128, 128, 0.5, 1)
    with pytest.raises(E.InvalidArgument):
        E.gemm_compressed(t, torch.zeros(4, 64, dtype=torch.float16, device="cuda"))


@pytest.mark.slow
@pytest.mark.parametrize("rows,cols,tokens", [(9216, 36864, 16), (36864, 9216, 128), (9216, 9216, 2048)])
def test_gemm_opt66b_shapes(E, rows, cols, tokens):
    t, W = _synth(E, rows, cols, 0.5, rows + cols)
    X = _x(tokens, cols, tokens)
    y = E.gemm_compressed(t, X, index=E.build_rank_index(t.bitmap, 1024))
    gemm_check(y, W, X)


@pytest.mark.parametrize("rows,cols,tokens", [(128, 64, 16), (300, 1000, 70), (256, 4096, 256), (129, 2048, 600),
                                              (1024, 9216, 1000)])
def test_dense_gemm_matches_fp64_reference(E, rows, cols, tokens):
    """the cuBLAS-free dense consumer (and the second pass of large-token GEMMs)"""
    g = torch.Generator(device="cpu").manual_seed(rows + cols)
    W = ((torch.rand(rows, cols, generator=g) * 2 - 1).half()).cuda()
    X = _x(tokens, cols, tokens)
    w = E.DenseMatrix(rows, cols, E.Dtype.F16, W.reshape(-1).view(torch.uint8).clone())
    y = E.gemm(w, X)
    gemm_check(y, W, X)
    assert torch.equal(y, E.gemm(w, X))


@pytest.mark.parametrize("rows,cols,tokens,s", [(300, 1024, 500, 0.5), (512, 9216, 1024, 0.5), (96, 1000, 900, 0.3)])
def test_gemm_two_pass_large_tokens(E, rows, cols, tokens, s):
    """tokens > 384: gemm_compressed decompresses W once into the workspace and
    runs the dense tcgen05 GEMM; same contract (and same errors) as the fused path"""
    if cols % 128:
        t, W = _oracle_tensor(E, rows, cols, s, rows + cols, values_offset=2)
    else:
        t, W = _synth(E, rows, cols, s, rows + cols)
    X = _x(tokens, cols, cols)
    y = E.gemm_compressed(t, X)
    gemm_check(y, W, X)
    y2 = E.gemm_compressed(t, X, index=E.build_rank_index(t.bitmap, 1024))
    assert torch.equal(y, y2)
    bad = E.EndorTensor(rows, cols, E.Dtype.F16, t.bitmap, t.values[:-2], validate=False)
    with pytest.raises(E.CorruptionError):
        E.gemm_compressed(bad, X)


def _pinned_prefix(E, t):
    idx = E.build_rank_index(t.bitmap, 1024)
    h = torch.empty(idx.prefix.numel(), dtype=torch.int64, pin_memory=True)
    h.copy_(idx.prefix.to(torch.int64))
    return h


@pytest.mark.parametrize("tokens", [16, 500])
def test_pipeline_gemm_ops(E, tokens):
    """endor_pipeline_op.tokens > 1: the offload pipeline streams each op's
    compressed W from pinned host memory and runs the GEMM consumer on it
    (fused below the two-pass threshold, decompress + dense GEMM above);
    with and without a pinned load-time RankIndex (prefix1024_host)."""
    from paper_2406_11674_b200.pipeline import HostOp, OffloadPipeline, pinned_copy
    shapes = [(256, 2048), (128, 1024), (96, 1000)]
    ts, Ws = [], []
    for i, (r, c) in enumerate(shapes):
        if c % 128:
            t, W = _oracle_tensor(E, r, c, 0.5, 77 + i)
        else:
            t, W = _synth(E, r, c, 0.5, 77 + i)
        ts.append(t)
        Ws.append(W)
    Xs = [_x(tokens, t.cols, i) for i, t in enumerate(ts)]
    for with_prefix in (False, True):
        ops = [HostOp(t.rows, t.cols, 0, pinned_copy(t.bitmap.data), pinned_copy(t.values), t.nnz(), x=X,
                      y=torch.empty(tokens, t.rows, dtype=torch.float32, device="cuda"),
                      y_host=torch.empty(tokens * t.rows, dtype=torch.float32, pin_memory=True), tokens=tokens,
                      prefix1024=_pinned_prefix(E, t) if with_prefix else None)
               for t, X in zip(ts, Xs)]
        p = OffloadPipeline(0, max(t.element_count() for t in ts))
        p.run(ops, sync=True)
        st = p.stats()
        p.close()
        for o, W, X in zip(ops, Ws, Xs):
            gemm_check(o.y_host.reshape(tokens, -1).cuda(), W, X)
        assert st["h2d_bytes"] == sum(o.compressed_bytes for o in ops)
