"""decompress_chunked timing on fc1 at chunk 1024 / 2048 / 4096 / 8192
(development aid): back-to-back over two rotating copies (no L2 reuse),
CUDA events.  Usage: [ENDOR_LIB=...] python tools/chunked_time.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2406_11674_b200 import catalog, codec as E  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6550.0
w = E.synth_weight(9216, 36864, 7, device="cuda")
E.magnitude_prune(w, 0.5, inplace=True)
ts = [E.compress(w)]
ts.append(E.EndorTensor(ts[0].rows, ts[0].cols, ts[0].dtype, E.Bitmap(ts[0].bitmap.size(), ts[0].bitmap.data.clone()),
                        ts[0].values.clone(), validate=False, nnz=ts[0].nnz()))
alg = catalog.algorithmic_bytes(ts[0].element_count(), ts[0].nnz())
for cs in (1024, 2048, 4096, 8192):
    plans = [E.BatchPlan([t], indices=[E.build_rank_index(t.bitmap, cs)]) for t in ts]
    for p in plans:
        p.launch()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for r in range(20):
        plans[r % 2].launch()
    b.record()
    torch.cuda.synchronize()
    for p in plans:
        p.sync()
    ms = a.elapsed_time(b) / 20
    ok = torch.equal(plans[0].outs[0].data, w.data)
    print(json.dumps({"cs": cs, "ms": round(ms, 4), "frac": round(alg / ms / 1e6 / PEAK, 4), "bit_exact": ok}))
