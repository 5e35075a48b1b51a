"""One decompress_chunked call on fc1 (9216 x 36864 f16 @ 50 %) at a chosen
chunk size, for ncu captures (development aid).  Usage: python tools/chunked_one.py CS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_11674_b200 import codec as E  # noqa: E402

cs = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
w = E.synth_weight(9216, 36864, 7, device="cuda")
E.magnitude_prune(w, 0.5, inplace=True)
t = E.compress(w)
idx = E.build_rank_index(t.bitmap, cs)
for _ in range(3):
    out = E.decompress_chunked(t, idx)
torch.cuda.synchronize()
assert torch.equal(out.data, w.data)
print("ok", cs)
