"""Fused decompress -> GEMV across sparsity on fc1 (9216 x 36864), both
consumers (development aid): ENDOR_GV_SPARSE=0 (byte lanes, per-slot cost) or
=1 (set-bit walk, per-value cost); unset = the library's automatic choice.
Prints ms per call and the max error vs the dense GEMV."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_11674_b200 import _lib, catalog, codec as E  # noqa: E402

dev = torch.device("cuda", 0)
L = _lib.lib()
rows, cols = 9216, 36864
res = {}
for s in (0.3, 0.5, 0.6, 0.7, 0.75, 0.8, 0.9, 0.95):
    w = E.synth_weight(rows, cols, catalog.FC1_SEED, device=dev)
    E.magnitude_prune(w, s, inplace=True)
    t = E.compress(w)
    idx = E.build_rank_index(t.bitmap, 1024).prefix.contiguous()
    x = (torch.rand(cols, device=dev, generator=torch.Generator("cuda").manual_seed(1)) * 2 - 1).half()
    y = torch.empty(rows, dtype=torch.float32, device=dev)
    v = t.view()
    ws = E.workspace(t.element_count(), dev)
    st = torch.cuda.current_stream().cuda_stream

    def run():
        E.check(L.endor_cuda_gemv_compressed(C.byref(v), idx.data_ptr(), x.data_ptr(), y.data_ptr(), None,
                                             ws.data_ptr(), ws.numel(), st))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        run()
    b.record()
    torch.cuda.synchronize()
    E.sync_status(ws, dev)
    ms = a.elapsed_time(b) / 20
    ref = E.gemv(w, x)
    err = (y - ref).abs().max().item() / max(ref.abs().max().item(), 1e-30)
    res[s] = {"ms": round(ms, 4), "rel_err": err, "compressed_gbs": round(t.compressed_bytes() / (ms * 1e-3) / 1e9, 1)}
    print(s, res[s], flush=True)
    del w, t
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/fused_sweep_%s.json" % os.environ.get("ENDOR_GV_SPARSE", "auto"), "w"), indent=1)
