"""compress (codec.hpp:97-126) timing on fc1 and one OPT-66B layer (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_11674_b200 import catalog, codec as E  # noqa: E402

for label, ops in (("fc1", [(9216, 36864)]), ("opt-66b layer", [(o.rows, o.cols) for o in catalog.model_catalog("opt-66b").ops])):
    ws = []
    for i, (r, c) in enumerate(ops):
        w = E.synth_weight(r, c, 7 + i, device="cuda")
        E.magnitude_prune(w, 0.5, inplace=True)
        ws.append(w)
    for w in ws:
        E.compress(w)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for rep in range(5):
        for w in ws:
            t = E.compress(w)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    dense = sum(w.size_bytes() for w in ws)
    print(f"{label}: compress {ms:.3f} ms per pass ({dense / ms / 1e6:.0f} dense-GB/s, includes the host sync per call)")
