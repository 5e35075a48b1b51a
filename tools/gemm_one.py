"""One fused GEMM launch on an OPT-66B shape (for ncu captures; development aid).
Usage: python tools/gemm_one.py [shape] [tokens] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_11674_b200 import codec as E  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "fc1"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 128
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
rows, cols = {"qkv": (9216, 9216), "fc1": (9216, 36864), "fc2": (36864, 9216)}[shape]
w = E.synth_weight(rows, cols, 1, device="cuda")
E.magnitude_prune(w, 0.5, inplace=True)
t = E.compress(w)
idx = E.build_rank_index(t.bitmap, 1024)
X = (torch.rand(T, cols, device="cuda") * 2 - 1).half()
for _ in range(reps):
    y = E.gemm_compressed(t, X, index=idx)
torch.cuda.synchronize()
print("ok", y.shape)
