"""decompress_chunk_into through the host-buffer C ABI (the entry point the
C++ drop-in `endor::cuda::decompress_chunk_into` binds, codec.hpp:191-201):
only chunk k's bytes move in either direction, every chunk is bit-exact
against the oracle, exactly chunk k's region of dst is written (the 0xAB
sentinel, test_codec.cpp:181-200), the reference's error order holds
(check_index tail CORRUPTION, then BOUNDS, then invalid_argument,
codec.hpp:193-197), and host threads may fan the calls out concurrently
(codec.hpp:203-204).
"""
import ctypes as C
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

CORRUPTION, BOUNDS, INVALID = 2, 3, 4


@pytest.fixture(scope="module")
def L(cuda_lib):
    return cuda_lib


def prefix_of(bm, n, cs):
    bits = np.unpackbits(bm, bitorder="little")[:n].astype(np.uint64)
    cum = np.concatenate([[0], np.cumsum(bits, dtype=np.uint64)])
    chunks = (n + cs - 1) // cs if n else 0
    return np.ascontiguousarray(cum[np.arange(chunks, dtype=np.int64) * cs], dtype=np.uint64)


def call(L, rows, cols, eb, bm, vals, nnz, cs, pre, k, dst, dst_bytes=None):
    dt = 0 if eb == 2 else 1  # Dtype::F16 = 0, Dtype::I8 = 1 (codec.hpp)
    return L.endor_cuda_decompress_chunk_into_host(
        rows, cols, dt, bm.ctypes.data, vals.ctypes.data if len(vals) else None, nnz, cs,
        pre.ctypes.data if len(pre) else None, len(pre), k, dst.ctypes.data,
        dst.size if dst_bytes is None else dst_bytes)


CASES = [(1, 1, 64), (3, 8197, 4096), (17, 12345, 1 << 20), (1000, 333, 100), (64, 8192, 8192),
         (5, 2049, 2000), (2, 4096, 64), (40, 3000, 777)]


@pytest.mark.parametrize("eb", [1, 2])
def test_every_chunk_bit_exact_and_isolated(L, eb):
    for i, (rows, cols, cs) in enumerate(CASES):
        for zf in (0.0, 0.6, 1.0):
            n = rows * cols
            w = O.random_dense(rows, cols, eb, 40 + 7 * i + int(10 * zf), zf)
            bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
            pre = prefix_of(bm, n, cs)
            full = np.full(n * eb, 0xAB, np.uint8)
            for k in range(len(pre)):
                dst = np.full(n * eb, 0xAB, np.uint8)
                assert call(L, rows, cols, eb, bm, vals, nnz, cs, pre, k, dst) == 0, L.endor_cuda_last_error_string()
                b, e = k * cs * eb, min((k + 1) * cs, n) * eb
                assert dst[b:e].tobytes() == w[b:e].tobytes(), (rows, cols, cs, zf, k)
                assert (dst[:b] == 0xAB).all() and (dst[e:] == 0xAB).all(), (rows, cols, cs, k)
                assert call(L, rows, cols, eb, bm, vals, nnz, cs, pre, k, full) == 0
            assert full.tobytes() == w.tobytes()


def test_error_order(L):
    rows, cols, eb, cs = 40, 3000, 2, 4096
    n = rows * cols
    w = O.random_dense(rows, cols, eb, 9, 0.5)
    bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
    pre = prefix_of(bm, n, cs)
    dst = np.zeros(n * eb, np.uint8)
    bad_tail = pre.copy()
    bad_tail[-1] += 1
    # the tail's CORRUPTION outranks BOUNDS and the destination-size check
    assert call(L, rows, cols, eb, bm, vals, nnz, cs, bad_tail, 0, dst) == CORRUPTION
    assert call(L, rows, cols, eb, bm, vals, nnz, cs, bad_tail, len(pre), dst) == CORRUPTION
    assert call(L, rows, cols, eb, bm, vals, nnz, cs, bad_tail, 0, dst, n * eb - 2) == CORRUPTION
    assert call(L, rows, cols, eb, bm, vals, nnz, cs, pre, len(pre), dst) == BOUNDS
    assert call(L, rows, cols, eb, bm, vals, nnz, cs, pre, 0, dst, n * eb - 2) == INVALID
    assert call(L, rows, cols, eb, bm, vals, nnz, cs, pre[:-1], 0, dst) == CORRUPTION  # does not cover
    # entries that would read past the values: beyond nnz, or a window that runs out
    for k, v in ((3, nnz + 1), (3, 2 ** 40), (len(pre) - 2, nnz - 5)):
        bad = pre.copy()
        bad[k] = v
        assert call(L, rows, cols, eb, bm, vals, nnz, cs, bad, k, dst) == CORRUPTION, (k, v)
    # the session is healthy afterwards
    for k in range(len(pre)):
        assert call(L, rows, cols, eb, bm, vals, nnz, cs, pre, k, dst) == 0
    assert dst.tobytes() == w.tobytes()


def test_threads_fan_out(L):
    """Host threads decompress disjoint chunks of one tensor into one buffer
    concurrently (each thread has its own device session and stream)."""
    rows, cols, eb, cs = 512, 4099, 2, 65536
    n = rows * cols
    w = O.random_dense(rows, cols, eb, 3, 0.5)
    bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
    pre = prefix_of(bm, n, cs)
    dst = np.full(n * eb, 0xAB, np.uint8)
    errs = []

    def run(t, T):
        torch.cuda.set_device(0)
        for k in range(t, len(pre), T):
            st = call(L, rows, cols, eb, bm, vals, nnz, cs, pre, k, dst)
            if st:
                errs.append((k, st))

    ts = [threading.Thread(target=run, args=(t, 6)) for t in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs
    assert dst.tobytes() == w.tobytes()


def test_device_chunk_into_threads_fan_out(L):
    """The device-pointer decompress_chunk_into from several Python threads on
    one tensor and one output (each thread gets its own workspace)."""
    from paper_2406_11674_b200 import codec as E
    rows, cols, eb, cs = 300, 5000, 2, 32768
    w = O.random_dense(rows, cols, eb, 21, 0.5)
    bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
    t = E.EndorTensor(rows, cols, E.Dtype.F16, E.Bitmap(rows * cols, data=torch.from_numpy(bm.copy()).cuda()),
                      torch.from_numpy(vals.copy()).cuda(), validate=False, nnz=nnz)
    idx = E.build_rank_index(t.bitmap, cs)
    out = torch.zeros(rows * cols * eb, dtype=torch.uint8, device="cuda")
    errs = []

    def run(tid, T):
        try:
            torch.cuda.set_device(0)
            for k in range(tid, idx.chunk_count(), T):
                E.decompress_chunk_into(t, idx, k, out)
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    ts = [threading.Thread(target=run, args=(i, 4)) for i in range(4)]
    for x in ts:
        x.start()
    for x in ts:
        x.join()
    torch.cuda.synchronize()
    assert not errs, errs
    assert out.cpu().numpy().tobytes() == w.tobytes()


def test_short_lived_threads_release_their_sessions(L):
    """Each host thread owns its device buffers, pinned staging and stream;
    they are released when the thread exits, so fanning calls out over
    short-lived threads does not accumulate device memory."""
    rows, cols, eb, cs = 64, 16384, 2, 1 << 18
    n = rows * cols
    w = O.random_dense(rows, cols, eb, 5, 0.5)
    bm, vals, nnz, _ = O.compress(w, rows, cols, eb)
    pre = prefix_of(bm, n, cs)
    dst = np.zeros(n * eb, np.uint8)

    def one(k):
        torch.cuda.set_device(0)
        assert call(L, rows, cols, eb, bm, vals, nnz, cs, pre, k, dst) == 0

    def wave():
        ts = [threading.Thread(target=one, args=(k % len(pre),)) for k in range(16)]
        for x in ts:
            x.start()
        for x in ts:
            x.join()

    wave()  # warm-up: the runtime's own per-thread state
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(5):
        wave()
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    # 80 sessions of ~1.7 MiB device buffers each would be > 100 MiB
    assert free0 - free1 < 32 << 20, (free0 - free1) >> 20
    assert dst.tobytes() == w.tobytes()
