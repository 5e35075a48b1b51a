"""decompress_chunk_into over HOST buffers, fanned out per chunk -- the
reference's own usage pattern (codec.hpp:191-204; its CPU baseline in
bench.py --impl reference runs exactly this over 16 threads) -- through the
C ABI the C++ drop-in binds (endor_cuda_decompress_chunk_into_host).
Development aid.

fc1 (9216 x 36864 f16 @ 50 %) generated on the GPU and copied to host memory,
chunk 2^20; every chunk once, single thread and T threads; dense GB/s.
Usage: python tools/chunk_into_host_time.py [--threads 16] [--max-chunks N]
"""
import argparse
import ctypes as C
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2406_11674_b200 import _lib, codec as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=16)
    ap.add_argument("--max-chunks", type=int, default=0, help="time only the first N chunks (slow builds)")
    ap.add_argument("--cs", type=int, default=1 << 20)
    a = ap.parse_args()
    L = _lib.lib()
    rows, cols, cs = 9216, 36864, a.cs
    w = E.synth_weight(rows, cols, 7, device="cuda")
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    bm = t.bitmap.data.cpu().numpy()
    vals = t.values.cpu().numpy()
    dense = w.data.view(torch.uint8).cpu().numpy().reshape(-1)
    idx = E.build_rank_index(t.bitmap, cs)
    pre = np.ascontiguousarray(idx.prefix.cpu().numpy().astype(np.uint64))
    n = rows * cols
    chunks = len(pre) if not a.max_chunks else min(a.max_chunks, len(pre))
    dst = np.ones(n * 2, np.uint8)  # touched: no first-touch page faults inside the timing

    def one(k):
        st = L.endor_cuda_decompress_chunk_into_host(rows, cols, 0, bm.ctypes.data, vals.ctypes.data, t.nnz(), cs,
                                                     pre.ctypes.data, len(pre), k, dst.ctypes.data, dst.size)
        assert st == 0, L.endor_cuda_last_error_string()

    for k in range(min(chunks, 4)):  # session warm-up (device buffers, pinned staging, stream)
        one(k)
    res = {"workload": "fc1 9216x36864 f16 @50 %, host buffers", "chunk": cs, "chunks_timed": chunks}
    t0 = time.perf_counter()
    for k in range(chunks):
        one(k)
    dt = time.perf_counter() - t0
    res["single_thread"] = {"s": round(dt, 4), "us_per_call": round(dt / chunks * 1e6, 1),
                            "dense_gbs": round(min(chunks * cs, n) * 2 / dt / 1e9, 2)}

    def run(tid, T):
        torch.cuda.set_device(0)
        for k in range(tid, chunks, T):
            one(k)

    for T in (a.threads,):
        ts = [threading.Thread(target=run, args=(i, T)) for i in range(T)]
        t0 = time.perf_counter()
        for x in ts:
            x.start()
        for x in ts:
            x.join()
        dt = time.perf_counter() - t0
        res[f"threads_{T}"] = {"s": round(dt, 4), "dense_gbs": round(min(chunks * cs, n) * 2 / dt / 1e9, 2)}
    if chunks == len(pre):
        res["bit_exact"] = bool((dst == dense).all())
    print(json.dumps(res))


if __name__ == "__main__":
    main()
