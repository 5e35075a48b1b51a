"""A/B of the offload pipeline on one OPT-66B layer (development aid): fused
decompress -> GEMV vs materialised W (decompress + dense GEMV), alternated
several times; prints per-run layer ms and H2D GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_11674_b200 import catalog  # noqa: E402
from paper_2406_11674_b200 import codec as E  # noqa: E402
from paper_2406_11674_b200.pipeline import HostOp, OffloadPipeline, pinned_copy  # noqa: E402

dev = torch.device("cuda", 0)
spec = catalog.model_catalog("opt-66b")
ops, nmax = [], 0
for i, op in enumerate(spec.ops):
    w = E.synth_weight(op.rows, op.cols, catalog.op_seed(0, i), device=dev)
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    del w
    x = (torch.rand(op.cols, device=dev) * 2 - 1).half()
    ops.append(HostOp(op.rows, op.cols, 0, pinned_copy(t.bitmap.data), pinned_copy(t.values), t.nnz(), x=x,
                      y=torch.empty(op.rows, dtype=torch.float32, device=dev),
                      y_host=torch.empty(op.rows, dtype=torch.float32, pin_memory=True)))
    nmax = max(nmax, op.rows * op.cols)
    torch.cuda.empty_cache()
mat = [HostOp(h.rows, h.cols, 0, h.bitmap, h.values, h.nnz, x=h.x, y=h.y, y_host=h.y_host, materialize=True)
       for h in ops]
depth = int(os.environ.get("RING", "2"))
pipe = OffloadPipeline(0, nmax, ring_depth=depth)
steps = 5
for name, o in (("fused", ops), ("materialized", mat)):
    pipe.run(o, sync=True)
for rep in range(3):
    for name, o in (("fused", ops), ("materialized", mat)):
        pipe.run(o * steps, sync=True)
        st = pipe.stats()
        print(f"{name:13s} layer_ms {st['total_ms'] / steps:8.3f}  h2d {st['h2d_bytes'] / st['h2d_ms'] / 1e6:6.2f} GB/s"
              f"  compute/layer {st['decompress_ms'] / steps + st['gemv_ms'] / steps:6.3f} ms"
              f"  exposed {st['exposed_compute_ms']:.3f} ms", flush=True)
pipe.close()
