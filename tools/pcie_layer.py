"""One OPT-66B decoder layer (six f16 @ 50 % ops) through the offload pipeline
from pinned host memory, for an ncu range-replay capture of the PCIe counters
over the NVTX range endor_pipeline_run (development aid):

  ncu --replay-mode app-range --nvtx --nvtx-include "endor_pipeline_run/" \\
      --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,gpu__time_duration.sum python tools/pcie_layer.py

The first run is a warm-up; both runs are sync (the NVTX range spans the
whole execution)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_11674_b200 import codec as E  # noqa: E402
from paper_2406_11674_b200.pipeline import HostOp, OffloadPipeline, pinned_copy  # noqa: E402

dev = torch.device("cuda", 0)
ops, nmax, comp = [], 0, 0
shapes = [(9216, 9216)] * 4 + [(9216, 36864), (36864, 9216)]
for i, (r, c) in enumerate(shapes):
    w = E.synth_weight(r, c, 1000 + i, device=dev)
    E.magnitude_prune(w, 0.5, inplace=True)
    t = E.compress(w)
    del w
    x = (torch.rand(c, device=dev) * 2 - 1).half()
    ops.append(HostOp(r, c, 0, pinned_copy(t.bitmap.data), pinned_copy(t.values), t.nnz(), x=x,
                      y=torch.empty(r, dtype=torch.float32, device=dev),
                      y_host=torch.empty(r, dtype=torch.float32, pin_memory=True)))
    nmax = max(nmax, r * c)
    comp += ops[-1].compressed_bytes
    del t
torch.cuda.empty_cache()
p = OffloadPipeline(0, nmax)
for _ in range(2):
    p.run(ops, sync=True)
st = p.stats()
print(f"compressed bytes {comp}, total {st['total_ms']:.3f} ms, h2d {st['h2d_ms']:.3f} ms, "
      f"{st['h2d_bytes'] / (st['h2d_ms'] * 1e-3) / 1e9:.2f} GB/s (events)")
p.close()
