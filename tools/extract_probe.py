"""Selective decompression (extract_rows / extract_cols, codec.hpp:239-297) on
OPT-66B fc1 at several selection fractions, through the raw C ABI (development
aid).  Algorithmic bytes: the counting pass over the whole bitmap (n/8) + the
selected rows' bitmap and values (rows), or every row's bitmap and at most one
32-byte value sector per selected value, capped at all values (cols) + the
dense output."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_11674_b200 import _lib, catalog, codec as E  # noqa: E402

dev = torch.device("cuda", 0)
L = _lib.lib()
PEAK = 6549.8
rows, cols = 9216, 36864
w = E.synth_weight(rows, cols, catalog.FC1_SEED, device=dev)
E.magnitude_prune(w, 0.5, inplace=True)
t = E.compress(w)
v = t.view()
n = rows * cols
ws = E.workspace(n, dev)
st = torch.cuda.current_stream().cuda_stream
g = torch.Generator(device="cpu").manual_seed(0)
res = {}
KINDS = os.environ.get("KINDS", "rows,cols").split(",")
FRACS = [float(f) for f in os.environ.get("FRACS", "0.001,0.01,0.05,0.25,0.5").split(",")]
for frac in FRACS:
    for kind in KINDS:
        m = rows if kind == "rows" else cols
        k = max(1, int(m * frac))
        sel = torch.randperm(m, generator=g)[:k].sort().values.to(torch.int64).to(dev)
        out = torch.empty((k * cols if kind == "rows" else rows * k) * 2 + 16, dtype=torch.uint8, device=dev)
        fn = L.endor_cuda_extract_rows if kind == "rows" else L.endor_cuda_extract_cols

        def run():
            E.check(fn(C.byref(v), sel.data_ptr(), k, out.data_ptr(), ws.data_ptr(), ws.numel(), st))
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        E.sync_status(ws, dev)
        dense_out = (k * cols if kind == "rows" else rows * k) * 2
        if kind == "rows":
            touched = k * cols // 8 + int(t.nnz() * k / rows) * 2
        else:  # every row's bits + at most one 32-byte value sector per selected value
            touched = n // 8 + min(t.nnz() * 2, int(t.nnz() * frac) * 32)
        alg = n // 8 + touched + dense_out
        ref = w.data.view(torch.float16).reshape(rows, cols)
        got = out[:dense_out].view(torch.float16).reshape((k, cols) if kind == "rows" else (rows, k))
        exact = bool(torch.equal(got, ref[sel] if kind == "rows" else ref[:, sel]))
        res[f"{kind}_{frac}"] = {"selected": k, "ms": round(ms, 4), "alg_bytes": alg,
                                 "frac_of_hbm_roofline": round(alg / (ms * 1e-3) / 1e9 / PEAK, 3),
                                 "bit_exact": exact}
        print(kind, frac, res[f"{kind}_{frac}"], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/extract_probe%s.json" % os.environ.get("ENDOR_EXTRACT_COLS_RPC", ""), "w"), indent=1)
