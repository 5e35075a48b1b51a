"""Randomised differential test of every device entry point against the CPU
oracle (development aid; test infrastructure like tests/, it imports oracle/).

  python tools/fuzz.py [seconds] [seed]

Shapes up to FUZZ_MAX_ELEMS elements (default 4M; 1..6000 per side), both dtypes, zero fractions
0..1 incl. the extremes, block-structured masks, odd value/bitmap offsets,
and every API: decompress, decompress_chunked (chunk 64..8192), chunk_into,
build_rank_index, extract_rows/cols, compress, fused GEMV (f16, cols % 1024
== 0) and dequant.  Prints the first mismatch and exits 1, else a summary."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2406_11674_b200 import codec as E  # noqa: E402

dev = torch.device("cuda", 0)


def dev_bytes(a, off):
    buf = torch.zeros(a.size + off + 64, dtype=torch.uint8, device=dev)
    v = buf[off: off + a.size]
    if a.size:
        v.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return v


MAX_ELEMS = int(os.environ.get("FUZZ_MAX_ELEMS", "4000000"))


def make(rng):
    eb = int(rng.choice([1, 2]))
    if rng.random() < 0.25:
        cols = int(rng.choice([1024, 2048, 3072, 8192, 9216]))
        rows = int(rng.integers(1, max(2, MAX_ELEMS // cols)))
    else:
        side = int(MAX_ELEMS ** 0.5 * 3)
        rows, cols = int(rng.integers(1, side)), int(rng.integers(1, side))
        while rows * cols > MAX_ELEMS:
            rows = max(1, rows // 2)
    zf = float(rng.choice([0.0, 1.0, rng.random()]))
    w = O.random_dense(rows, cols, eb, int(rng.integers(1 << 62)), zf)
    if rng.random() < 0.2:  # block structure: zero whole random row / column bands
        m = w.reshape(rows, cols * eb)
        r0 = int(rng.integers(0, rows))
        m[r0: r0 + int(rng.integers(1, rows + 1))] = 0
    return rows, cols, eb, w


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 120
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    t_end, n = time.time() + secs, 0
    while time.time() < t_end:
        rows, cols, eb, w = make(rng)
        bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
        t = E.EndorTensor(rows, cols, E.Dtype.F16 if eb == 2 else E.Dtype.I8,
                          E.Bitmap(rows * cols, data=dev_bytes(bm, 0)), dev_bytes(vals, int(rng.integers(0, 16))),
                          validate=False, nnz=nnz)
        want = w.tobytes()
        case = (rows, cols, eb, nnz)
        assert E.decompress(t).bytes() == want, ("decompress", case)
        cs = 64 << int(rng.integers(0, 8))
        idx = E.build_rank_index(t.bitmap, cs)
        pref = np.zeros(max(idx.chunk_count(), 1), np.uint64)
        O.lib().or_rank_index(bm, rows * cols, cs, pref)
        assert np.array_equal(idx.prefix.cpu().numpy().astype(np.uint64), pref[: idx.chunk_count()]), ("index", case, cs)
        assert E.decompress_chunked(t, idx).bytes() == want, ("chunked", case, cs)
        if idx.chunk_count():
            k = int(rng.integers(0, idx.chunk_count()))
            buf = torch.full((rows * cols * eb,), 0xAB, dtype=torch.uint8, device=dev)
            E.decompress_chunk_into(t, idx, k, buf)
            got = buf.cpu().numpy()
            lo, hi = k * cs * eb, min(rows * cols, (k + 1) * cs) * eb
            assert got[lo:hi].tobytes() == want[lo:hi], ("chunk_into", case, cs, k)
            assert (got[:lo] == 0xAB).all() and (got[hi:] == 0xAB).all(), ("chunk_into range", case, cs, k)
        full = w.reshape(rows, cols * eb)
        rsel = sorted(set(rng.integers(0, rows, int(rng.integers(0, min(rows, 40) + 1))).tolist()))
        assert E.extract_rows(t, rsel).bytes() == full[rsel].tobytes(), ("extract_rows", case)
        csel = sorted(set(rng.integers(0, cols, int(rng.integers(0, min(cols, 3000) + 1))).tolist()))
        wv = w.view(np.uint16 if eb == 2 else np.uint8).reshape(rows, cols)
        assert E.extract_cols(t, csel).bytes() == np.ascontiguousarray(wv[:, csel]).tobytes(), ("extract_cols", case)
        dense = E.DenseMatrix(rows, cols, t.dtype, dev_bytes(w, 0))
        tc = E.compress(dense)
        assert tc.nnz() == nnz and tc.bitmap.data.cpu().numpy().tobytes() == bm.tobytes(), ("compress", case)
        if eb == 2 and cols % 1024 == 0:
            x = (torch.rand(cols, device=dev) * 2 - 1).half()
            ref = torch.from_numpy(wv.view(np.float16).astype(np.float32)).to(dev) @ x.float()
            y = E.gemv_compressed(t, x)
            assert (y - ref).abs().max().item() <= 1e-3 * ref.abs().max().item() + 1e-6, ("gemv_compressed", case)
        if eb == 2:
            q = E.quantize_values(t)
            qv = q.values.cpu().numpy()
            q_ref, s_ref = O.quantize_values(vals, nnz)
            assert qv.tobytes() == q_ref.tobytes(), ("quantize", case)
            st, dq = O.decompress_dequant(rows, cols, bm, q_ref, nnz, s_ref)
            assert E.decompress_dequant(q).bytes() == dq.tobytes(), ("dequant", case)
        n += 1
    torch.cuda.synchronize()
    print(f"fuzz ok: {n} random cases in {secs:.0f} s")


if __name__ == "__main__":
    main()
