"""Measure every BASELINE.json config on one B200 (bench.py covers config 2).

  1  fc1 9216x36864 @50% round trip: GPU compress + decompress (index-free and
     1024-index paths) vs the reference CPU decompress on this host
  3  Llama2-70B layer @50%, row-sharded for G = 1, 2, 4, 8: the per-GPU work of
     a G-GPU box (each GPU's shard set decompressed on this GPU; no exchange
     exists on the data path, so per-GPU time is the scaling-relevant number)
  4  sparsity sweep 16384^2, s = 0.3 .. 0.9, full matrix (G=1) and 1/8 row
     shard (per-GPU work at G=8)
  5  whole OPT-66B forward pass: 64 layers streamed through the offload
     pipeline from 64 distinct pinned host buffers (decompress + GEMV per op);
     G=1 (73 GB) and the per-GPU 1/8 row shard of every layer (G=8)

Usage: python tools/configs_bench.py [--out profiles/r01/configs.json] [--skip-pass]
Timing: CUDA events, warm-up, inputs >> L2 except where noted ("l2" key).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2406_11674_b200 import catalog, codec as E, shard as S  # noqa: E402
from paper_2406_11674_b200.pipeline import HostOp, OffloadPipeline, pinned_copy  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
DEV = torch.device("cuda", 0)


def make(rows, cols, seed, s, r0=0, r1=None):
    w = E.synth_weight(rows, cols, seed, device=DEV)
    if s > 0:
        E.magnitude_prune(w, s, inplace=True)
    r1 = rows if r1 is None else r1
    part = E.DenseMatrix(r1 - r0, cols, E.Dtype.F16, w.data[r0 * cols * 2: r1 * cols * 2])
    t = E.compress(part)
    return t


def time_plan(plan, steps=20, warmup=3):
    st = torch.cuda.Stream(device=DEV)
    for _ in range(warmup):
        plan.launch(st.cuda_stream)
    plan.sync(st.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(steps):
        plan.launch(st.cuda_stream)
    b.record(st)
    torch.cuda.synchronize()
    plan.sync(st.cuda_stream)
    return a.elapsed_time(b) / steps


def decomp_stats(tensors, label, steps=20):
    outs = [E.DenseMatrix.empty(t.rows, t.cols, E.Dtype.F16, DEV) for t in tensors]
    idx = [E.build_rank_index(t.bitmap, 1024) for t in tensors]
    n = sum(t.element_count() for t in tensors)
    alg = sum(catalog.algorithmic_bytes(t.element_count(), t.nnz()) for t in tensors)
    res = {"label": label, "elements": n, "dense_bytes": 2 * n, "alg_bytes": alg}
    for name, plan in (("decompress_chunked_idx1024", E.BatchPlan(tensors, outs, indices=idx)),
                       ("decompress", E.BatchPlan(tensors, outs))):
        ms = time_plan(plan, steps)
        res[name] = {"ms": round(ms, 4), "dense_gbs": round(2 * n / (ms * 1e-3) / 1e9, 1),
                     "frac_of_hbm_roofline": round(alg / (ms * 1e-3) / 1e9 / PEAK, 4)}
    # y = W x: fused decompress -> GEMV (one batched call, 1024 index) vs the
    # materialised path's dense GEMV (one batched launch over the dense W)
    if all(t.dtype == E.Dtype.F16 and t.cols % 1024 == 0 for t in tensors):
        xs = [(torch.rand(t.cols, device=DEV) * 2 - 1).half() for t in tensors]
        st = torch.cuda.Stream(device=DEV)

        def timed(fn, reps=steps):
            with torch.cuda.stream(st):
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                for _ in range(reps):
                    fn()
                b.record(st)
                torch.cuda.synchronize()
            return a.elapsed_time(b) / reps

        comp = sum(t.compressed_bytes() + (t.element_count() // 1024) * 8 + t.cols * 2 for t in tensors)
        import ctypes as C
        from paper_2406_11674_b200 import _lib
        L, P, nt = _lib.lib(), C.c_void_p, len(tensors)
        views = (_lib.TensorView * nt)(*[t.view() for t in tensors])
        pres = [ix.prefix.contiguous() for ix in idx]
        ys = [torch.empty(t.rows, dtype=torch.float32, device=DEV) for t in tensors]
        pa, xa, ya = ((P * nt)(*[v.data_ptr() for v in vs]) for vs in (pres, xs, ys))
        ws = torch.zeros(L.endor_cuda_workspace_bytes_batch(views, nt), dtype=torch.uint8, device=DEV)

        def fused():  # the C ABI call alone: asynchronous, no host sync
            E.check(L.endor_cuda_gemv_compressed_batch(views, pa, xa, ya, None, nt, ws.data_ptr(), ws.numel(),
                                                       st.cuda_stream))

        ms_f = timed(fused)
        E.check(L.endor_cuda_sync_status(ws.data_ptr(), st.cuda_stream))
        for o, t in zip(outs, tensors):
            E.decompress(t, out=o)
        ms_g = timed(lambda: E.gemv_batch(outs, xs))
        res["fused_gemv_idx1024"] = {"ms": round(ms_f, 4), "weight_gbs": round(2 * n / (ms_f * 1e-3) / 1e9, 1),
                                     "frac_of_hbm_roofline": round(comp / (ms_f * 1e-3) / 1e9 / PEAK, 4)}
        res["dense_gemv"] = {"ms": round(ms_g, 4), "frac_of_hbm_roofline": round(2 * n / (ms_g * 1e-3) / 1e9 / PEAK, 4)}
        res["decompress_then_gemv_ms"] = round(res["decompress_chunked_idx1024"]["ms"] + ms_g, 4)
    res["l2"] = "inputs larger than L2" if alg > 3 * 126e6 else "fits in L2 (launch-bound regime)"
    return res


def cfg1(out):
    from oracle import oracle as O
    rows, cols = 9216, 36864
    w = E.synth_weight(rows, cols, catalog.FC1_SEED, device=DEV)
    E.magnitude_prune(w, 0.5, inplace=True)
    torch.cuda.synchronize()
    t0 = time.time()
    t = E.compress(w)
    torch.cuda.synchronize()
    comp_ms = (time.time() - t0) * 1e3
    r = decomp_stats([t], "opt-66b fc1 9216x36864 @50%")
    back = E.decompress(t)
    r["round_trip_bit_exact"] = bool(torch.equal(back.data, w.data))
    r["compress_wall_ms"] = round(comp_ms, 2)
    # the reference's own decompress on this host (oracle/_ref)
    R = O.ref()
    if R is not None:
        import ctypes as C
        import numpy as np
        bm, vals = t.bitmap.data.cpu().numpy().copy(), t.values.cpu().numpy().copy()
        st = C.c_int(0)
        h = R.ref_tensor_new(rows, cols, 2, bm, vals, t.nnz(), C.byref(st))
        t1 = R.ref_decompress_timed(h, None, C.byref(st))
        cs = 1 << 20
        pref = np.zeros((rows * cols + cs - 1) // cs, np.uint64)
        R.ref_rank_index(bm, rows * cols, cs, pref)
        dst = np.ones(rows * cols * 2, np.uint8)
        tp = min(R.ref_decompress_parallel_timed(h, pref, cs, len(pref), os.cpu_count(), dst.ctypes.data, C.byref(st))
                 for _ in range(3))
        R.ref_tensor_free(h)
        r["reference_cpu"] = {"single_thread_decompress_s": round(t1, 3), "parallel_s": round(tp, 4),
                              "threads": os.cpu_count(),
                              "single_thread_dense_gbs": round(rows * cols * 2 / t1 / 1e9, 3),
                              "parallel_dense_gbs": round(rows * cols * 2 / tp / 1e9, 2)}
    out["config1_fc1_round_trip"] = r


def cfg3(out):
    spec = catalog.model_catalog("llama2-70b")
    res = []
    for G in (1, 2, 4, 8):
        ts = []
        for oi, op in enumerate(spec.ops):
            sh = S.row_shard(op.rows, op.cols, 0, G)
            ts.append(make(op.rows, op.cols, catalog.op_seed(0, oi), 0.5, sh.r0, sh.r1))
        r = decomp_stats(ts, f"llama2-70b layer, per-GPU shard at G={G}")
        r["G"] = G
        res.append(r)
        del ts
        torch.cuda.empty_cache()
    out["config3_llama2_70b_layer_row_sharded"] = res


def cfg4(out):
    res = []
    for s in catalog.SWEEP_SPARSITIES:
        for G in (1, 8):
            sh = S.row_shard(16384, 16384, 0, G)
            t = make(16384, 16384, catalog.sweep_seed(s), s, sh.r0, sh.r1)
            r = decomp_stats([t], f"16384^2 @ s={s}, G={G} per-GPU shard")
            r.update(sparsity=s, G=G)
            res.append(r)
            del t
        torch.cuda.empty_cache()
    out["config4_sparsity_sweep_16384"] = res


def cfg5(out, G):
    """64-layer offloaded pass: the six OPT-66B ops (their 1/G row shards) are
    generated once and copied into 64 distinct pinned buffers per op."""
    spec = catalog.model_catalog("opt-66b")
    base = []
    for oi, op in enumerate(spec.ops):
        sh = S.row_shard(op.rows, op.cols, 0, G)
        t = make(op.rows, op.cols, catalog.op_seed(0, oi), 0.5, sh.r0, sh.r1)
        base.append((t, sh))
    g = torch.Generator(device="cpu").manual_seed(5)
    xs = [((torch.rand(op.cols, generator=g) * 2 - 1).half()).to(DEV) for op in spec.ops]
    ys = [torch.empty(sh.rows, dtype=torch.float32, device=DEV) for _, sh in base]
    yh = [torch.empty(sh.rows, dtype=torch.float32, pin_memory=True) for _, sh in base]
    ops = []
    for layer in range(spec.num_layers):
        for k, (t, sh) in enumerate(base):
            ops.append(HostOp(sh.rows, sh.cols, 0, pinned_copy(t.bitmap.data), pinned_copy(t.values), t.nnz(),
                              x=xs[k], y=ys[k], y_host=yh[k]))
    nmax = max(t.element_count() for t, _ in base)
    pipe = OffloadPipeline(0, nmax, ring_depth=2)
    pipe.run(ops[: len(base)], sync=True)  # warm-up: one layer
    pipe.run(ops, sync=True)
    st = pipe.stats()
    pipe.close()
    comp = sum(h.compressed_bytes for h in ops)
    dense = sum(h.dense_bytes for h in ops)
    return {"G": G, "layers": spec.num_layers, "ops": len(ops), "pass_ms": round(st["total_ms"], 2),
            "layer_ms": round(st["total_ms"] / spec.num_layers, 3), "h2d_bytes": comp,
            "h2d_gbs": round(st["h2d_bytes"] / (st["h2d_ms"] * 1e-3) / 1e9, 2),
            "dense_gbs_e2e": round(dense / (st["total_ms"] * 1e-3) / 1e9, 1),
            "decompress_ms_total": round(st["decompress_ms"], 2), "gemv_ms_total": round(st["gemv_ms"], 2),
            "exposed_compute_ms": round(st["exposed_compute_ms"], 3),
            "note": "per-GPU share on this box's PCIe link (G GPUs would each stream their own shards)"}


def cfg_structured(out):
    """SURVEY.md 8(d) cross-check: per-tile density made uneven or structured.
    fc1 shape with the reference's N:M pruning (nm_prune 2:4 and 1:4, restated
    in the oracle, weight_gen.hpp:118-141) and with whole-row bands pruned
    (every other block of 64 rows empty, the rest 80 % dense)."""
    import numpy as np
    from oracle import oracle as O
    rows, cols = 9216, 36864
    w = E.synth_weight(rows, cols, catalog.FC1_SEED, device=DEV)
    host = w.data.view(torch.uint8).cpu().numpy()
    res = []
    for keep, m in ((2, 4), (1, 4)):
        pr = np.zeros_like(host)
        assert O.lib().or_nm_prune(rows, cols, 2, keep, m, host, pr) == 0
        d = E.DenseMatrix(rows, cols, E.Dtype.F16, torch.from_numpy(pr).to(DEV))
        res.append(decomp_stats([E.compress(d)], f"fc1 nm_prune {keep}:{m}"))
        print(json.dumps(res[-1]), flush=True)
    wb = E.synth_weight(rows, cols, catalog.FC1_SEED, device=DEV)
    E.magnitude_prune(wb, 0.2, inplace=True)
    band = wb.data.view(torch.uint8).reshape(rows, cols * 2)
    for r0 in range(0, rows, 128):
        band[r0: r0 + 64] = 0
    res.append(decomp_stats([E.compress(wb)], "fc1 64-row bands alternately empty / 80 % dense"))
    print(json.dumps(res[-1]), flush=True)
    out["structured_sparsity_fc1"] = res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "configs.json"))
    ap.add_argument("--skip-pass", action="store_true")
    ap.add_argument("--only", default="", help="comma list of: structured (write only these keys)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    out = {"device": torch.cuda.get_device_name(0), "hbm_peak_gbs": PEAK, "host_threads": os.cpu_count()}
    if args.only:
        if "structured" in args.only:
            cfg_structured(out)
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
        return
    cfg1(out)
    print(json.dumps(out["config1_fc1_round_trip"]), flush=True)
    cfg3(out)
    cfg4(out)
    cfg_structured(out)
    if not args.skip_pass:
        out["config5_opt66b_64_layer_pass"] = [cfg5(out, 8), cfg5(out, 1)]
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out)[:4000])


if __name__ == "__main__":
    main()
