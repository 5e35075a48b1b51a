"""Development timing of the fused decompress -> GEMV kernel on one OPT-66B
layer (six f16 ops @50%), HBM-resident: per-op fused calls, one batched fused
call (with / without a 1024-chunk RankIndex), and the dense GEMV alone.
Prints per-path ms and the HBM roofline fraction (algorithmic bytes: bitmap +
packed values (+ x, y) for fused; 2 B/weight for the dense GEMV)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_11674_b200 import _lib, catalog  # noqa: E402
from paper_2406_11674_b200 import codec as E  # noqa: E402

L = _lib.lib()
dev = torch.device("cuda", 0)
PEAK = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json"))).get("hbm_gbs", 6552.3)
ops = [(o.rows, o.cols) for o in catalog.model_catalog("opt-66b").ops]
ts, xs, ys, idx, dense = [], [], [], [], []
for i, (r, c) in enumerate(ops):
    w = E.synth_weight(r, c, 1000 + i, device=dev)
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    ts.append(t)
    dense.append(w)
    g = torch.Generator(device="cpu").manual_seed(i)
    xs.append(((torch.rand(c, generator=g) * 2 - 1).half()).to(dev))
    ys.append(torch.empty(r, dtype=torch.float32, device=dev))
    idx.append(E.build_rank_index(t.bitmap, 1024).prefix.contiguous())
views = (_lib.TensorView * len(ts))(*[t.view() for t in ts])
nws = L.endor_cuda_workspace_bytes_batch(views, len(ts))
ws = torch.zeros(nws, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
P = C.c_void_p
pre_arr = (P * len(ts))(*[p.data_ptr() for p in idx])
x_arr = (P * len(ts))(*[x.data_ptr() for x in xs])
y_arr = (P * len(ts))(*[y.data_ptr() for y in ys])


def fused_batch(with_idx):
    E.check(L.endor_cuda_gemv_compressed_batch(views, pre_arr if with_idx else None, x_arr, y_arr, None, len(ts),
                                               ws.data_ptr(), ws.numel(), st))


def fused_per_op():
    for k in range(len(ts)):
        E.check(L.endor_cuda_gemv_compressed(C.byref(views[k]), P(idx[k].data_ptr()), P(xs[k].data_ptr()),
                                             P(ys[k].data_ptr()), None, ws.data_ptr(), ws.numel(), st))


def dense_gemv():
    for k in range(len(ts)):
        E.gemv(dense[k], xs[k], ys[k])


U64 = C.c_uint64
g_rows = (U64 * len(ts))(*[r for r, c in ops])
g_cols = (U64 * len(ts))(*[c for r, c in ops])
g_w = (P * len(ts))(*[d.data.data_ptr() for d in dense])


def dense_gemv_batch():
    E.check(L.endor_cuda_gemv_batch(g_rows, g_cols, g_w, x_arr, y_arr, None, len(ts), st))


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


comp = sum(t.compressed_bytes() for t in ts)
dn = sum(r * c * 2 for r, c in ops)
res = {}
for name, fn, byts in (("fused_batch_idx", lambda: fused_batch(True), comp),
                       ("fused_batch_count", lambda: fused_batch(False), comp),
                       ("fused_per_op_idx", fused_per_op, comp),
                       ("dense_gemv", dense_gemv, dn),
                       ("dense_gemv_batch", dense_gemv_batch, dn)):
    ms = timeit(fn)
    res[name] = {"ms": round(ms, 4), "gbs": round(byts / ms / 1e6, 1), "frac": round(byts / ms / 1e6 / PEAK, 3)}
    print(name, res[name], flush=True)
E.sync_status(ws, dev)
# accuracy vs fp32 reference
fused_batch(True)
torch.cuda.synchronize()
worst = 0.0
for k, (r, c) in enumerate(ops):
    ref = dense[k].data.view(torch.float16).reshape(r, c).float() @ xs[k].float()
    worst = max(worst, float((ys[k] - ref).abs().max() / ref.abs().max()))
print("max rel err vs fp32 reference:", worst)
res["max_rel_err"] = worst
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/fused_bench.json", "w"))
