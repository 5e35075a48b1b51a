"""Per-GPU shard workloads of the multi-GPU configs (SURVEY.md 8(d) configs 3
and 4 at G = 8) timed with the L2 flushed between repetitions, plus the count
pass alone.  Measurement aid (VERDICT r1 "small shards >= 0.70").

Three timings per workload (CUDA events on the launching stream):
  flushed       -- before each repetition write a 512 MiB scratch buffer and
                   then READ it back (a sum), so the 126 MB L2 holds only clean
                   lines of scratch: the inputs are cold and the timed call does
                   not pay for write-backs of someone else's dirty lines (a
                   write-only flush leaves ~126 MB of dirty scratch in L2 that
                   the timed kernel must evict -- ~20 us of HBM write time,
                   which is most of a G = 8 shard's budget);
  flushed_dirty -- the write-only flush (the r01/r02a method, kept for
                   comparison);
  rotating      -- back-to-back calls over R distinct copies of the workload
                   (R copies > 2x L2), i.e. the steady state of a layer-after-
                   layer pass: inputs never hit in L2, and each call drains the
                   previous call's dirty output lines as it would in the pass;
  back_to_back  -- the same inputs repeatedly (partly L2-resident).

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
L2_BYTES = 126 << 20


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
    plans = plan if isinstance(plan, list) else [plan]
    plan = plans[0]
    with torch.cuda.stream(st):
        for p in plans:
            for _ in range(2):
                p.launch(st.cuda_stream, phase=phase)
    torch.cuda.synchronize()
    if flush == "rotating":
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = reps * len(plans)
        a.record(st)
        with torch.cuda.stream(st):
            for i in range(n):
                plans[i % len(plans)].launch(st.cuda_stream, phase=phase)
        b.record(st)
        torch.cuda.synchronize()
        for p in plans:
            p.sync(st.cuda_stream)
        return a.elapsed_time(b) / n
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
            if flush == "clean":
                scratch.sum(dtype=torch.int64)  # read back: L2 left holding clean lines
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
    # rotating copies: R distinct (inputs, outputs) sets with R * bytes > 2 x L2
    R = max(2, min(16, -(-2 * L2_BYTES // max(alg, 1))))
    rot_i, rot_n = [pi], [pn]
    res["rotating_copies"] = R
    for _ in range(R - 1):
        ct = [E.EndorTensor(t.rows, t.cols, t.dtype, E.Bitmap(t.bitmap.size(), t.bitmap.data.clone()),
                            t.values.clone(), validate=False, nnz=t.nnz()) for t in tensors]
        co = [E.DenseMatrix.empty(t.rows, t.cols, E.Dtype.F16, DEV) for t in tensors]
        rot_i.append(E.BatchPlan(ct, co, indices=idx))
        rot_n.append(E.BatchPlan(ct, co))
    for name, plan, rot, phase in (("chunked_idx1024", pi, rot_i, 0), ("decompress", pn, rot_n, 0),
                                   ("count_only", pn, rot_n, 1), ("expand_only", pn, rot_n, 2)):
        r = {}
        for mode, key in (("clean", "flushed"), (True, "flushed_dirty"), ("rotating", "rotating"),
                          (False, "back_to_back")):
            if mode == "rotating" and phase == 2:
                continue  # expand_only needs its count pass in front of every call
            ms = timed(rot if mode == "rotating" else plan, reps, mode, phase)
            byts = bm if phase == 1 else alg
            r[key] = {"ms": round(ms, 4), "frac": round(byts / (ms * 1e-3) / 1e9 / PEAK, 4)}
        res[name] = r
    del rot_i, rot_n
    # size-matched ceiling: a device-to-device copy moving the same number of
    # bytes (alg / 2 read + alg / 2 written), timed the same ways -- the
    # launch + pipeline-fill floor every kernel of this size pays
    half = alg // 2
    srcs = [torch.empty(half, dtype=torch.uint8, device=DEV) for _ in range(R)]
    dsts = [torch.empty(half, dtype=torch.uint8, device=DEV) for _ in range(R)]

    class _Copy:
        def __init__(self, k):
            self.k = k

        def launch(self, stream_ptr=None, phase=0):
            dsts[self.k].copy_(srcs[self.k])

        def sync(self, stream_ptr=None):
            pass

    cps = [_Copy(k) for k in range(R)]
    r = {}
    for mode, key in (("clean", "flushed"), ("rotating", "rotating")):
        ms = timed(cps if mode == "rotating" else cps[0], reps, mode, 0)
        r[key] = {"ms": round(ms, 4), "frac": round(alg / (ms * 1e-3) / 1e9 / PEAK, 4)}
    res["d2d_copy_same_bytes"] = r
    for name in ("chunked_idx1024", "decompress"):
        res[name]["frac_of_d2d_copy"] = {k: round(r[k]["ms"] / res[name][k]["ms"], 4) for k in ("flushed", "rotating")}
    del srcs, dsts
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
