"""Quick check of the one-launch (look-back) decompress: small / ragged / batched
cases vs the oracle, then the OPT-66B layer timing (development aid)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2406_11674_b200 import codec as E  # noqa: E402

dev = torch.device("cuda", 0)
for (r, c, eb, zf) in [(1, 1, 2, 0.5), (3, 8197, 2, 0.5), (64, 8192, 1, 0.3), (1000, 333, 2, 0.9), (17, 12345, 2, 0.0),
                       (2, 5, 2, 1.0), (300, 4096, 2, 0.5)]:
    w = O.random_dense(r, c, eb, r * 7 + c, zf)
    bm, vals, nnz, _ = O.compress(w, r, c, eb)
    t = E.EndorTensor(r, c, E.Dtype.F16 if eb == 2 else E.Dtype.I8, E.Bitmap.from_bytes(bm.tobytes(), r * c, device=dev),
                      torch.from_numpy(vals.copy()).to(dev))
    for rep in range(3):
        assert E.decompress(t).bytes() == w.tobytes(), (r, c, eb, zf, rep)
print("small ok", flush=True)
w = E.synth_weight(9216, 36864, 7, device=dev)
E.magnitude_prune(w, 0.5, inplace=True)
t = E.compress(w)
for rep in range(5):
    assert torch.equal(E.decompress(t).data, w.data)
torch.cuda.synchronize()
out = E.DenseMatrix.empty(9216, 36864, E.Dtype.F16, dev)
plan = E.BatchPlan([t], [out])
for _ in range(3):
    plan.launch()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    plan.launch()
b.record()
torch.cuda.synchronize()
plan.sync()
print("fc1 decompress one launch: %.4f ms" % (a.elapsed_time(b) / 20), flush=True)
assert torch.equal(out.data, w.data)
# corrupted: popcount != nnz
bad = E.EndorTensor(t.rows, t.cols, t.dtype, t.bitmap, t.values[:-2], validate=False, nnz=t.nnz() - 1)
try:
    E.decompress(bad)
    raise SystemExit("expected CorruptionError")
except E.CorruptionError:
    pass
assert torch.equal(E.decompress(t).data, w.data)
print("lb smoke ok")
# batches with tensor boundaries inside 4-tile blocks
for shapes in ([(3, 8192), (1, 8192), (5, 8191), (2, 100)], [(1, 5)] * 9 + [(64, 8192)], [(9216, 9216)] * 4):
    ws_, ts_ = [], []
    for i, (r, c) in enumerate(shapes):
        if r * c > 10 ** 6:
            w = E.synth_weight(r, c, 50 + i, device=dev)
            E.magnitude_prune(w, 0.5, inplace=True)
            ws_.append(w.bytes())
            ts_.append(E.compress(w))
            continue
        w = O.random_dense(r, c, 2, 900 + i, 0.4)
        bm, vals, nnz, _ = O.compress(w, r, c, 2)
        ws_.append(w.tobytes())
        ts_.append(E.EndorTensor(r, c, E.Dtype.F16, E.Bitmap.from_bytes(bm.tobytes(), r * c, device=dev),
                                 torch.from_numpy(vals.copy()).to(dev)))
    for rep in range(3):
        outs = E.decompress_batch(ts_)
        assert [o.bytes() for o in outs] == ws_, shapes
print("batch ok")
