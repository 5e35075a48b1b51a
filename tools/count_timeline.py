"""Per-CTA phase timeline of count_kernel (development aid).  Needs a build
with -DENDOR_CTA_TIMING (tools/build_variant.sh timing -DENDOR_CTA_TIMING):
  ENDOR_LIB=tools/_build/libendor_timing.so python tools/count_timeline.py
Stamps: 0 CTA start, 1 after griddepcontrol.wait, 2 first block landed,
3 streaming done, 4 after the done-counter atomic, 5 last CTA's base scan done."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_2406_11674_b200 import _lib, catalog, codec as E  # noqa: E402
from small_shards import shard_of  # noqa: E402

DEV = torch.device("cuda", 0)
L = _lib.lib()
L.endor_debug_count_times.argtypes = [C.c_void_p, C.c_int]


def run(label, tensors):
    plan = E.BatchPlan(tensors)
    L.endor_debug_count_times((C.c_ulonglong * (8 * 4096))(), 0)
    st = torch.cuda.current_stream()
    for rep in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.launch(st.cuda_stream, phase=1)
        b.record()
        torch.cuda.synchronize()
    n = 4096
    buf = (C.c_ulonglong * (8 * n))()
    L.endor_debug_count_times(buf, n)
    t = np.array(buf, dtype=np.float64).reshape(n, 8)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    q = lambda c: [round(float(np.percentile(rel[:, c], p)), 2) for p in (0, 50, 100)]
    last = rel[rel[:, 5] > 0]
    print(json.dumps({"label": label, "ctas": len(t), "event_us": round(a.elapsed_time(b) * 1e3, 2),
                      "start_min_med_max": q(0), "pdl_wait_done": q(1), "first_block": q(2),
                      "stream_done": q(3), "atomic_done": q(4),
                      "last_cta_done": [round(float(x), 2) for x in last[:, 5]]}), flush=True)
    L.endor_debug_count_times  # keep


opt = catalog.model_catalog("opt-66b")
ts = [shard_of(op.rows, op.cols, catalog.op_seed(0, i), 0.5, 0, 1) for i, op in enumerate(opt.ops)]
run("opt-66b layer", ts)
del ts
spec = catalog.model_catalog("llama2-70b")
ts = [shard_of(op.rows, op.cols, catalog.op_seed(0, i), 0.5, 0, 8) for i, op in enumerate(spec.ops)]
run("llama2-70b G=8 shard", ts)
