"""Fused-GEMM time only (development aid for variant A/B runs):
python tools/gemm_time.py shape T [T ...]; ENDOR_LIB selects a variant build."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_11674_b200 import codec as E  # noqa: E402

shape = sys.argv[1]
rows, cols = {"qkv": (9216, 9216), "fc1": (9216, 36864), "fc2": (36864, 9216)}[shape]
w = E.synth_weight(rows, cols, 1, device="cuda")
E.magnitude_prune(w, 0.5, inplace=True)
t = E.compress(w)
idx = E.build_rank_index(t.bitmap, 1024)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
out = []
for T in [int(x) for x in sys.argv[2:]]:
    X = (torch.rand(T, cols, device="cuda") * 2 - 1).half()
    ts = []
    for _ in range(7):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        E.gemm_compressed(t, X, index=idx)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    out.append(f"T={T}: {ts[3]:.4f} ms ({2.0 * rows * cols * T / ts[3] / 1e9:.0f} TFLOP/s)")
print(os.path.basename(os.environ.get("ENDOR_LIB", "default")), shape, "; ".join(out))
