"""Every kernel of the library once on small shapes, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  Checks
results against the oracle as it goes, so a sanitizer run is also a parity run.

  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2406_11674_b200 import codec as E  # noqa: E402
from paper_2406_11674_b200 import storage as S  # noqa: E402
from paper_2406_11674_b200.pipeline import HostOp, OffloadPipeline, pinned_copy  # noqa: E402

dev = torch.device("cuda", 0)


def tensor(rows, cols, eb, seed, zf, offset=0):
    w = O.random_dense(rows, cols, eb, seed, zf)
    bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
    b = torch.zeros(len(bm) + 32, dtype=torch.uint8, device=dev)[: len(bm)]
    b.copy_(torch.from_numpy(bm))
    vb = torch.zeros(len(vals) + 64, dtype=torch.uint8, device=dev)[offset: offset + len(vals)]
    if len(vals):
        vb.copy_(torch.from_numpy(vals))
    t = E.EndorTensor(rows, cols, E.Dtype.F16 if eb == 2 else E.Dtype.I8, E.Bitmap(rows * cols, data=b), vb,
                      validate=False, nnz=nnz)
    return w, t


checks = 0
for (rows, cols, eb, zf, off) in [(2, 2, 2, 0.5, 0), (37, 1000, 2, 0.5, 2), (64, 2048, 2, 0.3, 6),
                                  (9, 4096, 1, 0.6, 1), (300, 1024, 2, 0.9, 10)]:
    w, t = tensor(rows, cols, eb, rows + cols, zf, off)
    assert E.decompress(t).bytes() == w.tobytes()                                  # count + TMA expand
    for cs in (64, 1024, 2048, 4096, 8192):
        idx = E.build_rank_index(t.bitmap, cs)                                     # scan_kernel
        assert E.decompress_chunked(t, idx).bytes() == w.tobytes()                 # fallback / fast / coarse
        buf = torch.zeros(t.dense_bytes(), dtype=torch.uint8, device=dev)
        for k in range(idx.chunk_count()):
            E.decompress_chunk_into(t, idx, k, buf)                                # partial-range expand
        assert buf.cpu().numpy().tobytes() == w.tobytes()
    sel = sorted({0, rows // 2, rows - 1})
    assert E.extract_rows(t, sel).bytes() == w.reshape(rows, cols * eb)[sel].tobytes()
    csel = sorted({0, cols // 3, cols - 1})
    got = E.extract_cols(t, csel).bytes()
    ref = w.view(np.uint16 if eb == 2 else np.uint8).reshape(rows, cols)[:, csel].tobytes()
    assert got == ref
    if eb == 2:
        dw = E.decompress(t)
        assert E.compress(dw).values.cpu().numpy().tobytes() == t.values.cpu().numpy().tobytes()
        x = (torch.rand(cols, device=dev) * 2 - 1).half()
        y = E.gemv(dw, x)                                                          # dense GEMV
        ref = torch.from_numpy(w.view(np.float16).reshape(rows, cols).astype(np.float32)).to(dev) @ x.float()
        assert (y - ref).abs().max().item() <= 1e-3 * ref.abs().max().item() + 1e-6
        if cols % 1024 == 0:
            yf = E.gemv_compressed(t, x)                                           # fused (count + flatten)
            assert (yf - ref).abs().max().item() <= 1e-3 * ref.abs().max().item() + 1e-6
            yi = E.gemv_compressed(t, x, index=E.build_rank_index(t.bitmap, 1024))
            assert torch.equal(yf, yi)
        q = E.quantize_values(t)                                                   # absmax + quantize
        E.decompress_dequant(q)                                                    # fused dequant expand
    checks += 1

# adversarial, validation-passing 1024 indices (garbage allowed, out-of-bounds not)
wa, ta = tensor(64, 4096, 2, 5, 0.5, 2)
ga = E.build_rank_index(ta.bitmap, 1024).prefix.cpu().numpy().astype(np.int64)
rng = np.random.default_rng(0)
for _ in range(5):
    bad = ga.copy()
    for k in range(1, len(bad) - 1):
        bad[k] = int(rng.integers(bad[k - 1], min(bad[k - 1] + 1024, bad[k + 1]) + 1))
    try:
        E.decompress_chunked(ta, E.RankIndex(1024, torch.from_numpy(bad).to(dev)))
    except E.CorruptionError:
        pass

# coarse (2048 / 4096 / 8192) indices: every wrong entry is reported, never an out-of-bounds access
for cs in (2048, 4096, 8192):
    gc = E.build_rank_index(ta.bitmap, cs).prefix.cpu().numpy().astype(np.int64)
    for _ in range(4):
        bad = np.sort(rng.integers(0, int(ta.nnz()) + 1, size=len(gc))).astype(np.int64)
        bad[0] = 0
        for v in (bad, gc + np.arange(len(gc)), np.full_like(gc, 10 ** 12)):
            try:
                E.decompress_chunked(ta, E.RankIndex(cs, torch.from_numpy(v).to(dev)))
            except E.CorruptionError:
                pass
    assert E.decompress_chunked(ta, E.RankIndex(cs, torch.from_numpy(gc).to(dev))).bytes() == wa.tobytes()

# the fused GEMV's set-bit consumer (density <= 0.2), odd value offset
w9, t9 = tensor(48, 4096, 2, 99, 0.9, 3)
x9 = (torch.rand(4096, device=dev) * 2 - 1).half()
y9 = E.gemv_compressed(t9, x9)
ref9 = torch.from_numpy(w9.view(np.float16).reshape(48, 4096).astype(np.float32)).to(dev) @ x9.float()
assert (y9 - ref9).abs().max().item() <= 1e-3 * ref9.abs().max().item() + 1e-6
d9 = E.dequantize_values(E.quantize_values(t9))
assert d9.nnz() == t9.nnz()

# batched paths
ws = [tensor(40, 2048, 2, s, 0.5) for s in range(3)]
outs = E.decompress_batch([t for _, t in ws])
assert [o.bytes() for o in outs] == [w.tobytes() for w, _ in ws]
xs = [(torch.rand(2048, device=dev) * 2 - 1).half() for _ in ws]
E.gemv_compressed_batch([t for _, t in ws], xs)
E.gemv_batch([E.decompress(t) for _, t in ws], xs)

# fixtures
sw = E.synth_weight(64, 1024, 5, device=dev)
E.magnitude_prune(sw, 0.5, inplace=True)

# storage (+ GPU CRC) and the pipeline, host- and file-sourced
with tempfile.TemporaryDirectory() as d:
    w, t = tensor(33, 2048, 2, 7, 0.5)
    p = os.path.join(d, "t.endor")
    S.write_endor_file(t, p)
    got = S.read_endor_file(p, dev, verify=True)
    assert E.decompress(got).bytes() == w.tobytes()
    x = (torch.rand(2048, device=dev) * 2 - 1).half()
    e0 = torch.empty(0, dtype=torch.uint8)
    ops = [HostOp(33, 2048, 0, pinned_copy(t.bitmap.data), pinned_copy(t.values), t.nnz(), x=x,
                  y=torch.empty(33, dtype=torch.float32, device=dev)),
           HostOp(33, 2048, 0, e0, e0, t.nnz(), path=p, x=x, y=torch.empty(33, dtype=torch.float32, device=dev)),
           HostOp(33, 2048, 0, pinned_copy(t.bitmap.data), pinned_copy(t.values), t.nnz(), x=x,
                  y=torch.empty(33, dtype=torch.float32, device=dev), materialize=True)]
    pipe = OffloadPipeline(0, 33 * 2048)
    pipe.run(ops, sync=True)
    pipe.close()
    assert torch.equal(ops[0].y, ops[1].y)
# host-buffer decompress_chunk_into (pinned staging, per-thread stream), arbitrary chunk size
from paper_2406_11674_b200 import _lib  # noqa: E402
L = _lib.lib()
for rows, cols, cs in ((5, 2049, 2000), (40, 3000, 4096)):
    w = O.random_dense(rows, cols, 2, rows + cols, 0.5)
    bm, vals, nnz, _ = O.compress(w, rows, cols, 2)
    n = rows * cols
    bits = np.unpackbits(bm, bitorder="little")[:n].astype(np.uint64)
    cum = np.concatenate([[0], np.cumsum(bits, dtype=np.uint64)])
    pre = np.ascontiguousarray(cum[np.arange((n + cs - 1) // cs) * cs], dtype=np.uint64)
    dst = np.zeros(n * 2, np.uint8)
    for k in range(len(pre)):
        assert L.endor_cuda_decompress_chunk_into_host(rows, cols, 0, bm.ctypes.data, vals.ctypes.data, nnz, cs,
                                                       pre.ctypes.data, len(pre), k, dst.ctypes.data, dst.size) == 0
    assert dst.tobytes() == w.tobytes()
    checks += 1
torch.cuda.synchronize()
print(f"sanitize smoke ok ({checks} shapes)")
