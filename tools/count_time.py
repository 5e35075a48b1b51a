"""Count-pass timing (development aid): count_kernel alone (BatchPlan phase 1)
on one OPT-66B layer and on a Llama2-70B G=8 shard, back-to-back over R
rotating copies (inputs never L2-resident), plus the whole no-index decompress.
Usage: [ENDOR_LIB=...] python tools/count_time.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

from paper_2406_11674_b200 import catalog, codec as E  # noqa: E402
from small_shards import PEAK, shard_of, timed  # noqa: E402

DEV = torch.device("cuda", 0)


def run(label, tensors, R):
    plans = [E.BatchPlan(tensors)]
    for _ in range(R - 1):
        ct = [E.EndorTensor(t.rows, t.cols, t.dtype, E.Bitmap(t.bitmap.size(), t.bitmap.data.clone()),
                            t.values.clone(), validate=False, nnz=t.nnz()) for t in tensors]
        plans.append(E.BatchPlan(ct))
    bm = sum(t.bitmap_bytes() for t in tensors)
    alg = sum(catalog.algorithmic_bytes(t.element_count(), t.nnz()) for t in tensors)
    c = timed(plans, 20, "rotating", 1)
    d = timed(plans, 20, "rotating", 0)
    out = {"label": label, "bitmap_bytes": bm, "count_us": round(c * 1e3, 2),
           "count_gbs": round(bm / c / 1e6, 1), "count_frac": round(bm / c / 1e6 / PEAK, 4),
           "decompress_us": round(d * 1e3, 2), "decompress_frac": round(alg / d / 1e6 / PEAK, 4)}
    print(json.dumps(out), flush=True)


opt = catalog.model_catalog("opt-66b")
ts = [shard_of(op.rows, op.cols, catalog.op_seed(0, i), 0.5, 0, 1) for i, op in enumerate(opt.ops)]
run("opt-66b layer", ts, 2)
del ts
torch.cuda.empty_cache()
spec = catalog.model_catalog("llama2-70b")
ts = [shard_of(op.rows, op.cols, catalog.op_seed(0, i), 0.5, 0, 8) for i, op in enumerate(spec.ops)]
run("llama2-70b G=8 shard", ts, 4)
