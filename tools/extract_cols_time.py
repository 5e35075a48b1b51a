"""extract_cols on fc1 (9216 x 36864 f16 @ 50 %) at several column fractions,
L2 flushed (fill + read back) before each call, CUDA events (development aid).
Usage: python tools/extract_cols_time.py"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2406_11674_b200 import _lib, codec as E  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
DEV = torch.device("cuda", 0)


def main():
    L = _lib.lib()
    rows, cols = 9216, 36864
    w = E.synth_weight(rows, cols, 7, device=DEV)
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    dense = w.data.view(torch.int16).reshape(rows, cols)
    v = t.view()
    n = rows * cols
    ws = E.workspace(n, DEV)
    st = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=DEV)
    bm_bytes, val_bytes = (n + 7) // 8, t.nnz() * 2
    for frac in (0.005, 0.01, 0.02, 0.05, 0.1, 0.25, 0.5, 1.0):
        k = max(1, int(cols * frac))
        sel = torch.arange(0, cols, cols // k, device=DEV, dtype=torch.int64)[:k].contiguous()
        ob = torch.empty(k * rows * 2 + 16, dtype=torch.uint8, device=DEV)
        ts = []
        for r in range(12):
            flush.fill_(r)
            flush.sum(dtype=torch.int64)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            assert L.endor_cuda_extract_cols(C.byref(v), sel.data_ptr(), k, ob.data_ptr(), ws.data_ptr(),
                                             ws.numel(), st) == 0
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        E.sync_status(ws, DEV)
        ms = sorted(ts)[len(ts) // 2]
        ok = torch.equal(ob[: k * rows * 2].view(torch.int16).reshape(rows, k), dense[:, sel])
        alg = bm_bytes + min(val_bytes, int(k * rows * 0.5) * 32) + k * rows * 2
        print(json.dumps({"frac": frac, "ncols": k,
                          "ms": round(ms, 4), "frac_of_peak": round(alg / (ms * 1e-3) / 1e9 / PEAK, 3),
                          "bit_exact": ok}), flush=True)


if __name__ == "__main__":
    main()
