"""Per-GPU work of bench.py at N=8 (eight layers' 1/8 row shards = 48 tensors)
decompressed with 6, 16 (or more) tensors per launch (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_11674_b200 import catalog, codec as E, shard as S  # noqa: E402

dev = torch.device("cuda", 0)
G = int(os.environ.get("G", "8"))
spec = catalog.model_catalog("opt-66b")
ts = []
for layer in range(G):
    for oi, op in enumerate(spec.ops):
        sh = S.row_shard(op.rows, op.cols, 0, G)
        w = E.synth_weight(op.rows, op.cols, catalog.op_seed(layer, oi), device=dev)
        E.magnitude_prune(w, 0.5, inplace=True)
        part = E.DenseMatrix(sh.rows, op.cols, E.Dtype.F16, w.data[sh.r0 * op.cols * 2: sh.r1 * op.cols * 2])
        ts.append(E.compress(part))
        del w, part
    torch.cuda.empty_cache()
outs = [E.DenseMatrix.empty(t.rows, t.cols, E.Dtype.F16, dev) for t in ts]
idx = [E.build_rank_index(t.bitmap, 1024) for t in ts]
alg = sum(catalog.algorithmic_bytes(t.element_count(), t.nnz()) for t in ts)
st = torch.cuda.Stream()
for per in [int(x) for x in os.environ.get("PER", "6,16").split(",")]:
    plans = [E.BatchPlan(ts[i:i + per], outs[i:i + per], indices=idx[i:i + per]) for i in range(0, len(ts), per)]
    for _ in range(3):
        for p in plans:
            p.launch(st.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(10):
        for p in plans:
            p.launch(st.cuda_stream)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"G={G} {len(ts)} tensors, {per} per launch ({len(plans)} launches): {ms:.4f} ms per step, "
          f"{alg / ms / 1e6:.1f} GB/s = {alg / ms / 1e6 / 6549.8:.3f} of peak", flush=True)
