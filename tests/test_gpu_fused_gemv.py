"""§8(f) row 1: fused decompress -> GEMV (y = W x from the compressed W).
Floating point: checked ELEMENT-WISE against a float64 reference GEMV over the
reference-exact decompressed W (conftest.gemv_check: every row within 1e-3 of
sum_j |W_ij x_j|, and within 1e-3 relative wherever y_ref is not dominated by
cancellation -- north star's 1e-3 relative tolerance), and bit-identical
across runs (deterministic order)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import gemv_check  # noqa: E402
from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E(cuda_lib):
    from paper_2406_11674_b200 import codec
    return codec


@pytest.mark.parametrize("rows,cols,s", [(1, 1024, 0.5), (37, 2048, 0.0), (300, 9216, 0.5), (64, 36864, 0.9),
                                         (1024, 8192, 0.3), (300, 9216, 0.85), (7, 1024, 0.97), (40, 4096, 0.999)])
def test_fused_gemv_matches_fp32_reference(E, rows, cols, s):
    w = E.synth_weight(rows, cols, rows * 31 + cols, device="cuda")
    if s > 0:
        E.magnitude_prune(w, s, inplace=True)
    t = E.compress(w)
    g = torch.Generator(device="cpu").manual_seed(cols)
    x = ((torch.rand(cols, generator=g) * 2 - 1).half()).cuda()
    Wd = w.data.view(torch.float16).reshape(rows, cols)
    y = E.gemv_compressed(t, x)
    gemv_check(y, Wd, x)
    y2 = E.gemv_compressed(t, x, index=E.build_rank_index(t.bitmap, 1024))
    assert torch.equal(y, y2)              # same partials, same order
    assert torch.equal(y, E.gemv_compressed(t, x))  # deterministic
    # and equal to the materialised path within fp32 rounding
    gemv_check(E.gemv(E.decompress(t), x), Wd, x)


def test_fused_gemv_rejects_unsupported(E):
    w = O.random_dense(4, 1000, 2, 1, 0.5)
    bm, vals, nnz, _ = O.compress(w, 4, 1000, 2)
    b = torch.zeros(len(bm) + 32, dtype=torch.uint8, device="cuda")[: len(bm)]
    b.copy_(torch.from_numpy(bm))
    v = torch.from_numpy(vals.copy()).cuda()
    t = E.EndorTensor(4, 1000, E.Dtype.F16, E.Bitmap(4000, data=b), v)
    with pytest.raises(E.InvalidArgument):  # cols % 1024 != 0
        E.gemv_compressed(t, torch.zeros(1000, dtype=torch.float16, device="cuda"))


def _layer(E, shapes, s, seed0):
    ts, ws, xs = [], [], []
    for i, (r, c) in enumerate(shapes):
        w = E.synth_weight(r, c, seed0 + i, device="cuda")
        if s > 0:
            E.magnitude_prune(w, s, inplace=True)
        ts.append(E.compress(w))
        ws.append(w)
        g = torch.Generator(device="cpu").manual_seed(seed0 + 100 + i)
        xs.append(((torch.rand(c, generator=g) * 2 - 1).half()).cuda())
    return ts, ws, xs


@pytest.mark.parametrize("with_index", [False, True])
def test_fused_gemv_batch_mixed_shapes(E, with_index):
    """One batched launch over ragged shapes (rows % 8 != 0, cols from 1 to 36
    segments, a sub-8-sub-tile tensor) equals the per-tensor fused path and the
    fp32 reference of the decompressed W."""
    shapes = [(37, 2048), (9, 36864), (300, 9216), (1, 1024), (64, 8192), (3, 3072)]
    ts, ws, xs = _layer(E, shapes, 0.5, 900)
    idx = [E.build_rank_index(t.bitmap, 1024) for t in ts] if with_index else None
    ys = E.gemv_compressed_batch(ts, xs, idx)
    for t, w, x, y in zip(ts, ws, xs, ys):
        gemv_check(y, w.data.view(torch.float16).reshape(t.rows, t.cols), x)
        assert torch.equal(y, E.gemv_compressed(t, x))  # same partials, same order


def test_fused_gemv_batch_detects_bad_index(E):
    ts, ws, xs = _layer(E, [(64, 2048), (16, 4096)], 0.5, 77)
    idx = [E.build_rank_index(t.bitmap, 1024) for t in ts]
    bad = idx[1].prefix.clone()
    bad[5] += 3  # a middle entry inconsistent with the bitmap
    idx[1] = E.RankIndex(1024, bad)
    with pytest.raises(E.CorruptionError):
        E.gemv_compressed_batch(ts, xs, idx)


def test_dense_gemv_batch_matches_fp32_reference(E):
    shapes = [(9216, 1024), (5, 36864), (1000, 9216), (33, 8)]
    ts, ws, xs = _layer(E, shapes, 0.3, 4242)
    ys = E.gemv_batch(ws, xs)
    for w, x, y in zip(ws, xs, ys):
        gemv_check(y, w.data.view(torch.float16).reshape(w.rows, w.cols), x)
        assert torch.equal(y, E.gemv(w, x))  # batched launch == single launch, bitwise


def test_pipeline_fused_matches_materialized(E):
    """The offload pipeline's default fused decompress -> GEMV and its
    materialised path (flags bit1) give the same y within fp32 rounding."""
    from paper_2406_11674_b200.pipeline import HostOp, OffloadPipeline, pinned_copy
    shapes = [(96, 2048), (40, 9216), (7, 1000)]  # the last one cannot fuse (cols % 1024)
    ts, ws, xs = _layer(E, shapes, 0.5, 31337)
    outs = {}
    for mat in (False, True):
        ops = [HostOp(t.rows, t.cols, 0, pinned_copy(t.bitmap.data), pinned_copy(t.values), t.nnz(), x=x,
                      y=torch.empty(t.rows, dtype=torch.float32, device="cuda"),
                      y_host=torch.empty(t.rows, dtype=torch.float32, pin_memory=True), materialize=mat)
               for t, x in zip(ts, xs)]
        p = OffloadPipeline(0, max(t.element_count() for t in ts))
        p.run(ops, sync=True)
        p.close()
        outs[mat] = [o.y_host.clone() for o in ops]
    for a, b, w, x in zip(outs[False], outs[True], ws, xs):
        Wd = w.data.view(torch.float16).reshape(w.rows, w.cols)
        gemv_check(a, Wd, x)
        gemv_check(b, Wd, x)


def test_fused_gemv_nonfinite_weights_stay_in_their_rows(E):
    """Raw-bit NaN / inf weights (legal in the format, test_codec.cpp:123-130)
    poison only their own row's y; every other row matches the fp32 reference
    (the gather never lets a neighbouring row's values into a product)."""
    rows, cols = 24, 2048
    w = E.synth_weight(rows, cols, 99, device="cuda")
    E.magnitude_prune(w, 0.5, inplace=True)
    wh = w.data.view(torch.float16).reshape(rows, cols)
    nz = (wh[0] != 0).nonzero()[0].item()
    wh[0, nz] = float("nan")
    nz5 = (wh[5] != 0).nonzero()[3].item()
    wh[5, nz5] = float("inf")
    t = E.compress(w)
    x = (torch.rand(cols, generator=torch.Generator().manual_seed(3)) + 0.5).half().cuda()  # finite, > 0
    y = E.gemv_compressed(t, x)
    assert torch.isnan(y[0]) and torch.isinf(y[5]) and y[5] > 0
    ok = torch.ones(rows, dtype=torch.bool, device="cuda")
    ok[0] = ok[5] = False
    assert torch.isfinite(y[ok]).all()
    gemv_check(y[ok], wh[ok], x)


@pytest.mark.parametrize("offset", [2, 6, 10, 14])
def test_fused_gemv_unaligned_values_buffer(E, offset):
    """The packed values may start at any 2-byte offset (the .endor layout puts
    them at 32 + ceil(n/8), file_io.hpp:32-36): the TMA windows' ragged ends are
    copied bytewise; results equal the aligned case bitwise."""
    rows, cols = 50, 3072
    w = E.synth_weight(rows, cols, 4242, device="cuda")
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    vb = t.values.numel()
    buf = torch.zeros(vb + 64, dtype=torch.uint8, device="cuda")
    buf[offset:offset + vb].copy_(t.values)
    tu = E.EndorTensor(rows, cols, E.Dtype.F16, t.bitmap, buf[offset:offset + vb], validate=False, nnz=t.nnz())
    x = (torch.rand(cols, generator=torch.Generator().manual_seed(1)) * 2 - 1).half().cuda()
    assert torch.equal(E.gemv_compressed(tu, x), E.gemv_compressed(t, x))
    assert torch.equal(E.gemv_compressed(tu, x, index=E.build_rank_index(t.bitmap, 1024)), E.gemv_compressed(t, x))


@pytest.mark.parametrize("mode", ["0", "1"])
def test_every_fused_case_under_each_consumer(cuda_lib, mode):
    """This file again with the consumer forced (ENDOR_GV_SPARSE=0: byte
    lanes, =1: set-bit walk) -- the library otherwise picks by density."""
    import os
    import subprocess
    import sys
    if os.environ.get("ENDOR_GV_SPARSE") is not None:
        pytest.skip("already forced")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ENDOR_GV_SPARSE=mode)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_fused_gemv.py"),
                        os.path.join(root, "tests", "test_gpu_density.py")],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
