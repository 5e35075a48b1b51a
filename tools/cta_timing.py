"""Per-CTA start/end times of expand_tma_kernel (development aid).

Needs a variant build with -DENDOR_CTA_TIMING:
  tools/build_variant.sh timing -DENDOR_CTA_TIMING
  ENDOR_LIB=tools/_build/libendor_timing.so python tools/cta_timing.py
Prints, for a small G=8 shard and a full layer: event time, first-start to
last-end span, CTA start spread, min/median/max CTA lifetime."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_11674_b200 import _lib, catalog, codec as E, shard as S  # noqa: E402

DEV = torch.device("cuda", 0)


def run(label, tensors, cs=1024):
    L = _lib.lib()
    outs = [E.DenseMatrix.empty(t.rows, t.cols, E.Dtype.F16, DEV) for t in tensors]
    idx = [E.build_rank_index(t.bitmap, cs) for t in tensors]
    plan = E.BatchPlan(tensors, outs, indices=idx)
    scratch = torch.empty(512 << 20, dtype=torch.uint8, device=DEV)
    res = []
    for rep in range(6):
        scratch.fill_(rep)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.launch(torch.cuda.current_stream().cuda_stream)
        b.record()
        torch.cuda.synchronize()
        buf = (C.c_ulonglong * (3 * 296))()
        L.endor_debug_cta_times(buf, 296)
        t = np.array(buf, dtype=np.float64).reshape(296, 3)
        t = t[t[:, 0] > 0]  # the grid is one CTA per SM: drop the unused slots
        st, en, sm = t[:, 0], t[:, 1], t[:, 2].astype(int)
        life = (en - st) / 1e3
        res.append({"event_us": round(a.elapsed_time(b) * 1e3, 2), "span_us": round((en.max() - st.min()) / 1e3, 2),
                    "start_spread_us": round((st.max() - st.min()) / 1e3, 2),
                    "life_us_min_med_max": [round(float(life.min()), 2), round(float(np.median(life)), 2),
                                            round(float(life.max()), 2)],
                    "slowest_cta": int(life.argmax()), "slowest_sm": int(sm[life.argmax()]),
                    "slow_ctas(>1.25 median)": [(int(i), int(sm[i]), round(float(life[i]), 1))
                                                for i in np.nonzero(life > 1.25 * np.median(life))[0]][:12],
                    "end_us_sorted_last5": [round(float(x), 1) for x in np.sort((en - st.min()) / 1e3)[-5:]],
                    "end_us_p10_p50_p90": [round(float(np.percentile((en - st.min()) / 1e3, q)), 1) for q in (10, 50, 90)]})
    print(json.dumps({"label": label, "reps": res[3:]}))
    if os.environ.get("CTA_DUMP"):
        order = np.argsort(sm)
        print(json.dumps({"label": label, "by_sm": [[int(sm[i]), int(i), round(float(life[i]), 1)] for i in order]}))


def main():
    L = _lib.lib()
    L.endor_debug_cta_times.argtypes = [C.c_void_p, C.c_int]
    if "--fc1" in sys.argv:  # fc1 alone at chunk 1024 and at the coarse 4096 (deriver path)
        w = E.synth_weight(9216, 36864, 7, device=DEV)
        E.magnitude_prune(w, 0.5, inplace=True)
        t = E.compress(w)
        del w
        run("fc1 cs=1024", [t], 1024)
        run("fc1 cs=4096", [t], 4096)
        return
    w = E.synth_weight(16384, 16384, 150, device=DEV)
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    del w
    run("16384^2 s=0.5 G=8 shard 0", [S.shard_tensor(t, S.row_shard(16384, 16384, 0, 8), copy=True)])
    del t
    spec = catalog.model_catalog("llama2-70b")
    ts = []
    for i, op in enumerate(spec.ops):
        w = E.synth_weight(op.rows, op.cols, catalog.op_seed(0, i), device=DEV)
        E.magnitude_prune(w, 0.5, inplace=True)
        tt = E.compress(w)
        del w
        ts.append(S.shard_tensor(tt, S.row_shard(op.rows, op.cols, 0, 8), copy=True))
    run("llama2-70b G=8 shard 0", ts)
    del ts
    torch.cuda.empty_cache()
    spec = catalog.model_catalog("opt-66b")
    ts = []
    for i, op in enumerate(spec.ops):
        w = E.synth_weight(op.rows, op.cols, catalog.op_seed(0, i), device=DEV)
        E.magnitude_prune(w, 0.5, inplace=True)
        ts.append(E.compress(w))
        del w
    run("opt-66b layer G=1", ts)


if __name__ == "__main__":
    main()
