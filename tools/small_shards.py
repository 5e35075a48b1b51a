"""Per-GPU shard workloads of the multi-GPU configs (SURVEY.md 8(d) configs 3
and 4 at G = 8) timed with the L2 flushed between repetitions, plus the count
pass alone.  Measurement aid (VERDICT r1 "small shards >= 0.70").

Each repetition: write a 512 MiB scratch buffer (evicts the 126 MB L2), then
events around ONE decompress call on the same stream.  Also reported: the
back-to-back figure (no flush) for comparison.

Usage: python tools/small_shards.py [--out FILE] [--reps N]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2406_11674_b200 import catalog, codec as E, shard as S  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
DEV = torch.device("cuda", 0)


def shard_of(rows, cols, seed, s, g, G):
    w = E.synth_weight(rows, cols, seed, device=DEV)
    if s > 0:
        E.magnitude_prune(w, s, inplace=True)
    t = E.compress(w)
    del w
    return S.shard_tensor(t, S.row_shard(rows, cols, g, G), copy=True)


def timed(plan, reps, flush, phase=0):
    st = torch.cuda.Stream(device=DEV)
    scratch = torch.empty(512 << 20, dtype=torch.uint8, device=DEV)
    for _ in range(3):
        plan.launch(st.cuda_stream, phase=phase)
    torch.cuda.synchronize()
    if not flush:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            plan.launch(st.cuda_stream, phase=phase)
        b.record(st)
        torch.cuda.synchronize()
        plan.sync(st.cuda_stream)
        return a.elapsed_time(b) / reps
    evs = []
    with torch.cuda.stream(st):
        for r in range(reps):
            scratch.fill_(r & 0xFF)
            if phase == 2:
                plan.launch(st.cuda_stream, phase=1)  # the count pass, untimed
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            plan.launch(st.cuda_stream, phase=phase)
            b.record(st)
            evs.append((a, b))
    torch.cuda.synchronize()
    plan.sync(st.cuda_stream)
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    return ts[len(ts) // 2]  # median


def measure(label, tensors, reps):
    outs = [E.DenseMatrix.empty(t.rows, t.cols, E.Dtype.F16, DEV) for t in tensors]
    idx = [E.build_rank_index(t.bitmap, 1024) for t in tensors]
    n = sum(t.element_count() for t in tensors)
    alg = sum(catalog.algorithmic_bytes(t.element_count(), t.nnz()) for t in tensors)
    bm = sum(t.bitmap_bytes() for t in tensors)
    res = {"label": label, "elements": n, "alg_bytes": alg}
    pi = E.BatchPlan(tensors, outs, indices=idx)
    pn = E.BatchPlan(tensors, outs)
    for name, plan, phase in (("chunked_idx1024", pi, 0), ("decompress", pn, 0), ("count_only", pn, 1),
                              ("expand_only", pn, 2)):
        r = {}
        for flush in (True, False):
            ms = timed(plan, reps, flush, phase)
            byts = bm if phase == 1 else alg
            r["flushed" if flush else "back_to_back"] = {"ms": round(ms, 4),
                                                          "frac": round(byts / (ms * 1e-3) / 1e9 / PEAK, 4)}
        res[name] = r
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    out = {"pdl": os.environ.get("ENDOR_PDL", "1"), "peak_gbs": PEAK, "rows": []}
    spec = catalog.model_catalog("llama2-70b")
    opt = catalog.model_catalog("opt-66b")
    for G in ((8,) if a.quick else (1, 8)):
        ts = [shard_of(op.rows, op.cols, catalog.op_seed(0, i), 0.5, 0, G) for i, op in enumerate(spec.ops)]
        out["rows"].append(measure(f"llama2-70b layer G={G} shard 0", ts, a.reps))
        del ts
        torch.cuda.empty_cache()
    ts = [shard_of(op.rows, op.cols, catalog.op_seed(0, i), 0.5, 0, 1) for i, op in enumerate(opt.ops)]
    out["rows"].append(measure("opt-66b layer G=1", ts, a.reps))
    del ts
    torch.cuda.empty_cache()
    for s in ((0.5, 0.9) if a.quick else (0.3, 0.5, 0.7, 0.9)):
        for G in (8,):
            t = shard_of(16384, 16384, 100 + round(100 * s), s, 0, G)
            out["rows"].append(measure(f"16384^2 s={s} G={G} shard 0", [t], a.reps))
            del t
            torch.cuda.empty_cache()
    txt = json.dumps(out, indent=1)
    print(txt)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt)


if __name__ == "__main__":
    main()
